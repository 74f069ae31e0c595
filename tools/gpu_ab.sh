# A/B of kernel variants: tools/gpu_ab.sh "base v1 v2" DEGREES [pytest -k expr]
# base = the in-tree libdg_b200.so; vN = variants/libdg_vN.so swapped in for its runs
set -u
vars=$1; degs=$2; kexpr=${3:-}
cp paper_1907_08492_b200/libdg_b200.so /tmp/libdg_base.so
for rep in 1 2; do
  for v in $vars; do
    if [ $v = base ]; then cp /tmp/libdg_base.so paper_1907_08492_b200/libdg_b200.so; else cp variants/libdg_$v.so paper_1907_08492_b200/libdg_b200.so; fi
    python bench.py --steps 5 --warmup 3 --quick --degrees $degs 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
  if l.startswith('{'):
    d=json.loads(l); print('$v', {p:(round(o['matvec_dofs_per_s']/1e9,1), round(o['cheby_step_dofs_per_s']/1e9,1), round(o['basis_change_gbs'])) for p,o in d['ops'].items()}, d['clocks']['sm_mhz'])
" >> gpurun_out/ab.log
  done
done
if [ -n "$kexpr" ]; then
  for v in $vars; do
    [ $v = base ] && continue
    cp variants/libdg_$v.so paper_1907_08492_b200/libdg_b200.so
    timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "$kexpr" > gpurun_out/pytest_ab_$v.log 2>&1; echo "pytest $v rc=$?" >> gpurun_out/ab.log
  done
fi
cp /tmp/libdg_base.so paper_1907_08492_b200/libdg_b200.so
