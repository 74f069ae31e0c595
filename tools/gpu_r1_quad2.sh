set -x
python -m pytest tests/test_gpu_quadrature.py tests/test_gpu_halo_loopback.py -x -q > gpurun_out/pytest_quad2.log 2>&1
echo "pytest rc=$?"
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --workload c3 > gpurun_out/bench_c3b.json 2> gpurun_out/bench_c3b.err
echo "c3 rc=$?"
python bench.py --steps 1 --warmup 0 --quick --workload c3 > gpurun_out/plain_c3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_quad -s 15 -c 1 -o gpurun_out/prof_quad2_c3 python bench.py --steps 1 --warmup 0 --quick --workload c3 > gpurun_out/ncu_quad2.log 2>&1
echo "ncu rc=$?"
