# A/B of environment settings: tools/gpu_env_ab.sh "VAR=a VAR=b ..." DEGREES
set -u
for rep in 1 2; do
  for kv in $1; do
    env $kv python bench.py --steps 5 --warmup 3 --quick --degrees $2 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
  if l.startswith('{'):
    d=json.loads(l); print('$kv', {p:(round(o['matvec_dofs_per_s']/1e9,1), round(o['cheby_step_dofs_per_s']/1e9,1)) for p,o in d['ops'].items()}, d['clocks']['sm_mhz'])
" >> gpurun_out/envab.log
  done
done
