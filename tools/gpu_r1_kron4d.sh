set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_halo_loopback.py -x -q > gpurun_out/pytest_k4d.log 2>&1
echo "pytest rc=$?"
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_k4d.json 2> gpurun_out/bench_k4d.err
echo "k4 rc=$?"
DG_K4_OUT=0 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_k4d0.json 2> gpurun_out/bench_k4d0.err
echo "k4 out0 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_kron4 -s 1 -c 2 -o gpurun_out/prof_k4d_p5 python bench.py --steps 1 --warmup 0 --quick --degrees 5 > gpurun_out/ncu_k4d.log 2>&1
echo "ncu rc=$?"
