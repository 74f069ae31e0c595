set -x
python -m pytest tests/test_gpu_halo_loopback.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_halo.log 2>&1
echo "pytest rc=$?"
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --workload c3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
echo "c3 rc=$?"
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --workload c2 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
echo "c2 rc=$?"
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --workload c5 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
echo "c5 rc=$?"
