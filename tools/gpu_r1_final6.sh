timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_final6.log 2>&1
echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke6.log 2>&1
echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench_c4_final6.json 2> gpurun_out/bench_c4_final6.err
echo "c4 rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_final6.json 2> gpurun_out/bench_ref_final6.err
echo "ref rc=$?"
