set -x
timeout 900 python -m pytest tests/test_gpu_quadrature.py -x -q > gpurun_out/pytest_q3.log 2>&1
echo "pytest rc=$?"
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --workload c3 > gpurun_out/bench_q3.json 2> gpurun_out/bench_q3.err
echo "c3 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_kron4<6, 2, 1' -s 1 -c 1 -o gpurun_out/prof_k4f_cheby python bench.py --steps 1 --warmup 0 --quick --degrees 5 > gpurun_out/ncu_k4f.log 2>&1
echo "ncu rc=$?"
du -sh gpurun_out/*.ncu-rep
