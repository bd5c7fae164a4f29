# A/B of library variants inside one gpurun call: bash tools/ab_lib.sh "" build/x/libhologen_b200.so ...
# ("" = the default in-tree library).  In-graph per-iteration time + bench kernel times.
for L in "$@"; do
  echo "lib=${L:-default}"
  if [ -n "$L" ]; then export HG_LIB=$PWD/$L; else unset HG_LIB; fi
  python tools/iter_time.py 4096 64 | cut -c1-200
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-ospr 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d['roofline'];print('  value', round(d['value'],1), 'row', round(r['row']['ms'],3), 'col', round(r['col']['ms'],3))"
done
unset HG_LIB
