set -u
mkdir -p gpurun_out/k3c
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_smoother_parity.py tests/test_gpu_halo_loopback.py tests/test_gpu_slab_transport.py -x -q -m gpu -k "p2 or -2- or p-2 or [2- or 2] or C1 or halo or slab or transport or single_cell" > gpurun_out/k3c/tests.log 2>&1; echo "tests rc=$?"
for v in 0 1; do DG_K3C=$v python bench.py --steps 5 --warmup 3 --quick --degrees 2 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
  if l.startswith('{'):
    d=json.loads(l); print('K3C=$v', {p:(round(o['matvec_dofs_per_s']/1e9,1), round(o['cheby_step_dofs_per_s']/1e9,1), round(o['cheby_frac_hbm'],3), round(o.get('cheby_fdm_step_dofs_per_s',0)/1e9,1)) for p,o in d['ops'].items()}, d['clocks']['sm_mhz'])
" >> gpurun_out/k3c/ab.log; done
cat gpurun_out/k3c/ab.log
