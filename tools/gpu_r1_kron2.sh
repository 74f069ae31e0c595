set -x
python -m pytest tests/test_gpu_parity.py tests/test_gpu_halo_loopback.py -x -q > gpurun_out/pytest_kron2.log 2>&1
echo "pytest rc=$?"
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_kron2.json 2> gpurun_out/bench_kron2.err
echo "bench rc=$?"
python bench.py --steps 1 --warmup 0 --quick --degrees 5 > gpurun_out/plain_p5c.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_kron -s 15 -c 2 -o gpurun_out/prof_kron2_p5 python bench.py --steps 1 --warmup 0 --quick --degrees 5 > gpurun_out/ncu_kron2.log 2>&1
echo "ncu rc=$?"
