timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "f32" > gpurun_out/pytest_f32.log 2>&1
echo "pytest rc=$?"
