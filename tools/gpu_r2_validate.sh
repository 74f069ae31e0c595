# Full validation on one B200: pytest -m gpu, smoke, default bench line
set -u
mkdir -p gpurun_out/val
python -m pytest tests -m gpu -q > gpurun_out/val/gputests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/val/gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/val/smoke.log 2>&1; echo "smoke rc=$?"; cat gpurun_out/val/smoke.log | tail -1
python bench.py > gpurun_out/val/bench_c4.json 2> gpurun_out/val/bench_c4.err; echo "bench rc=$?"
