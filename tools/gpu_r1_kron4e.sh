set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_k4e.log 2>&1
echo "pytest rc=$?"
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_k4e.json 2> gpurun_out/bench_k4e.err
echo "k4 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_kron4 -s 1 -c 2 -o gpurun_out/prof_k4e_p5 python bench.py --steps 1 --warmup 0 --quick --degrees 5 > gpurun_out/ncu_k4e.log 2>&1
echo "ncu rc=$?"
