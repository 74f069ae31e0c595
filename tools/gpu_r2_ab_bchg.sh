# basis-change A/B: tools/gpu_r2_ab_bchg.sh "base v1 env_X=1" DEGREES  -> gpurun_out/ab.log (GB/s per degree)
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
    d=json.loads(l); print('$v', {p:round(o['basis_change_gbs']) for p,o in d['ops'].items()}, d['clocks']['sm_mhz'])
" >> gpurun_out/ab.log
  done
done
cp /tmp/libdg_base.so paper_1907_08492_b200/libdg_b200.so
