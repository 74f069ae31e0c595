timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_final7.log 2>&1
echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke7.log 2>&1
echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench_c4_final7.json 2> gpurun_out/bench_c4_final7.err
echo "c4 rc=$?"
