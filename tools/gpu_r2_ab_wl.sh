# A/B of library variants on another workload: tools/gpu_r2_ab_wl.sh "base v1" WORKLOAD (c2|c3|c5)
set -u
vars=$1; wl=$2
cp paper_1907_08492_b200/libdg_b200.so /tmp/libdg_base.so
for rep in 1 2; do
  for v in $vars; do
    if [ $v = base ]; then cp /tmp/libdg_base.so paper_1907_08492_b200/libdg_b200.so; else cp variants/libdg_$v.so paper_1907_08492_b200/libdg_b200.so; fi
    python bench.py --workload $wl --steps 5 --warmup 3 --quick 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
  if l.startswith('{'):
    d=json.loads(l); print('$v', {p:(round(o['matvec_dofs_per_s']/1e9,2), round(o['cheby_step_dofs_per_s']/1e9,2), round(o['cheby_frac_hbm'],3)) for p,o in d['ops'].items()}, d['clocks']['sm_mhz'])
" >> gpurun_out/ab.log
  done
done
cp /tmp/libdg_base.so paper_1907_08492_b200/libdg_b200.so
