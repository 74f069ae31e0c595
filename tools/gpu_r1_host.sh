timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "host_buffers" > gpurun_out/pytest_host.log 2>&1
echo "pytest rc=$?"
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --degrees 5 > gpurun_out/bench_host.json 2> gpurun_out/bench_host.err
echo done
