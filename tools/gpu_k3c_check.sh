# k_kron3c checks on one B200: the p = 2 / C1 / slab parity subset, then an A/B of the given variants at p = 2
set -u
mkdir -p gpurun_out/k3c
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_smoother_parity.py tests/test_gpu_halo_loopback.py tests/test_gpu_slab_transport.py tests/test_gpu_user_penalty.py tests/test_gpu_variants.py -x -q -m gpu -k "p2 or -2- or p-2 or [2- or 2] or C1 or halo or slab or transport or single_cell or variant" > gpurun_out/k3c/tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/k3c/tests.log
rm -f gpurun_out/ab.log
[ -n "${1:-}" ] && bash tools/gpu_r2_ab.sh "$1" 2
cat gpurun_out/ab.log
