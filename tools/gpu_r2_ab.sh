# A/B of library variants on one box: tools/gpu_r2_ab.sh "base v1 v2" DEGREES [ENV-ASSIGNMENTS-PER-VARIANT via VAR_ENV_<name>]
# base = in-tree .so; vN = variants/libdg_vN.so.  Two rounds, bench --quick per variant -> gpurun_out/ab.log
set -u
vars=$1; degs=$2
cp paper_1907_08492_b200/libdg_b200.so /tmp/libdg_base.so
for rep in 1 2; do
  for v in $vars; do
    envs=""
    case $v in
      base) cp /tmp/libdg_base.so paper_1907_08492_b200/libdg_b200.so ;;
      env_*) cp /tmp/libdg_base.so paper_1907_08492_b200/libdg_b200.so; envs=$(echo ${v#env_} | tr '+' ' ') ;;
      *) cp variants/libdg_$v.so paper_1907_08492_b200/libdg_b200.so ;;
    esac
    env $envs python bench.py --steps 5 --warmup 3 --quick --degrees $degs 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
  if l.startswith('{'):
    d=json.loads(l); print('$v', {p:(round(o['matvec_dofs_per_s']/1e9,1), round(o['cheby_step_dofs_per_s']/1e9,1), round(o['cheby_frac_hbm'],3)) for p,o in d['ops'].items()}, 'frac', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])
" >> gpurun_out/ab.log
  done
done
cp /tmp/libdg_base.so paper_1907_08492_b200/libdg_b200.so
