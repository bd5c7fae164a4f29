# A/B of library variants on the seed kernel: GS seed ms per step and OSPR subframes/s.
# bash tools/ab_seed_ospr.sh "" build/x/libhologen_b200.so ...   ("" = the in-tree library)
for L in "$@"; do
  if [ -n "$L" ]; then export HG_LIB=$PWD/$L; else unset HG_LIB; fi
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d['roofline'];o=d['ospr'];print('lib=${L:-default}', 'gs', round(d['value'],1), 'seed_ms', round(r['seed_ms'],3), 'ospr', round(o['value'],1), 'ospr_seed_ms', round(o['roofline']['kernels']['seed']['ms'],3), 'single_job_ms', round(o['single_job']['ms_per_job'],3))"
done
unset HG_LIB
