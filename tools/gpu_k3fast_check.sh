set -u
mkdir -p gpurun_out/k3f
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_smoother_parity.py -x -q -m gpu -k "k3c_full_tiles or c4_full_size or p2 or 2-" > gpurun_out/k3f/tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/k3f/tests.log
rm -f gpurun_out/ab.log
bash tools/gpu_r2_ab.sh "k3nofast base" 2
cat gpurun_out/ab.log
