set -u
python -m pytest tests -m gpu -x -q -k "basis_change or smoke or chebyshev" > gpurun_out/pytest_bchg.log 2>&1; echo "pytest rc=$?"
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c4_bchg4.json 2> gpurun_out/bench_c4_bchg4.err; echo "c4 rc=$?"
DG_BCHG=1 python bench.py --steps 5 --warmup 3 --degrees 2,5,6,8 > gpurun_out/bench_c4_bchg1.json 2> gpurun_out/bench_c4_bchg1.err; echo "c4 old rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_bchg4 -s 2 -c 1 -o gpurun_out/prof_bchg4_p5 python bench.py --steps 1 --warmup 0 --quick --degrees 5 > gpurun_out/ncu_bchg.log 2>&1; echo "ncu rc=$?"
