timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "chebyshev" > gpurun_out/pytest_pre_odd.log 2>&1
echo "pytest rc=$?"
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --degrees 2,4,6,8 > gpurun_out/bench_pre_odd.json 2> gpurun_out/bench_pre_odd.err
echo done
