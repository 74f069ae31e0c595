# Transformed-residual Chebyshev step (KMODE_CHEBY_GLT): parity, then A/B against the direct step
set -u
mkdir -p gpurun_out/glt
python -m pytest tests/test_gpu_parity.py tests/test_gpu_smoother_parity.py -q -m gpu -k "cheby or smooth or pcg" -x > gpurun_out/glt/tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/glt/tests.log
python -m pytest tests/test_gpu_variants.py -q -m gpu -k "GLT" > gpurun_out/glt/variants.log 2>&1; echo "variants rc=$?"; tail -3 gpurun_out/glt/variants.log
rm -f gpurun_out/ab.log
bash tools/gpu_r2_ab.sh "base env_DG_CHEBY_GLT=0" "3,4,5,6,7,8"
cp gpurun_out/ab.log gpurun_out/glt/ab.log; cat gpurun_out/glt/ab.log
