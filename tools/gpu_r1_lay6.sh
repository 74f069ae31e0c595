timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_lay6.log 2>&1
echo "pytest rc=$?"
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_lay6.json 2> gpurun_out/bench_lay6.err
echo "bench rc=$?"
