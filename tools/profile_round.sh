#!/bin/bash
# Run on the GPU box (gpurun): the plain bench, the ncu launch list of the same
# command, and one ncu --set full capture of the fused passes at the bench's
# batch (64 targets of 4096^2).  Outputs land in gpurun_out/.
set -u
CMD="python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e"
$CMD > gpurun_out/prof_bench_plain.json 2> gpurun_out/prof_bench_plain.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    $CMD > gpurun_out/ncu_launches.log 2>&1 || echo "launch list rc=$?"
python tools/prof_gs.py 4096 64 2 > gpurun_out/prof_gs_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_row|k_col|k_seed|k_mt_jump" -s 1 -c 5 \
    -o gpurun_out/prof_full python tools/prof_gs.py 4096 64 2 > gpurun_out/ncu_full.log 2>&1
echo done
