timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "gpu_dot or apply_preconditioner or lanczos or pcg" > gpurun_out/pytest_solver.log 2>&1
echo "pytest rc=$?"
