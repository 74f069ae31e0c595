timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_quadrature.py -q -k "rows_longer or diagonal or chebyshev" > gpurun_out/pytest_rows.log 2>&1
echo "pytest rc=$?"
