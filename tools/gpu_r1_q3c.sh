timeout 900 python -m pytest tests/test_gpu_quadrature.py -x -q > gpurun_out/pytest_q3f.log 2>&1
echo "pytest rc=$?"
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --workload c3 > gpurun_out/bench_q3f.json 2> gpurun_out/bench_q3f.err
timeout 600 ncu --section LaunchStats --section Occupancy --section SpeedOfLight --clock-control none -k regex:k_quad3 -s 1 -c 1 python bench.py --steps 1 --warmup 0 --quick --workload c3 > gpurun_out/ncu_q3f.log 2>&1
echo done
