DG_K4_ALT=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_alt.log 2>&1
echo "pytest rc=$?"
for alt in 0 1; do
DG_K4_ALT=$alt timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --degrees 5,7 > gpurun_out/bench_alt$alt.json 2> gpurun_out/bench_alt$alt.err
done
echo done
