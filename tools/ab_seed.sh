# Seed-kernel A/B across library variants (inside one gpurun call).
for L in "$@"; do
  if [ -n "$L" ]; then export HG_LIB=$PWD/$L; else unset HG_LIB; fi
  timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d['roofline'];o=d['ospr'];print('${L:-default}', 'gs', round(d['value'],1), 'gs_seed', round(r['seed_ms'],3), 'ospr', round(o['value'],1), 'ospr_seed', round(o['roofline']['kernels']['seed']['ms'],3), 'single', round(o['single_job']['ms_per_job'],3))"
done
unset HG_LIB
