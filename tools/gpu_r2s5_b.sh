# Round 2 session 5, step B: new basis-change defaults (plane mode) -- tests, A/B, bench
set -u
mkdir -p gpurun_out/s5
python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py tests/test_gpu_mixed_precision.py tests/test_gpu_smoother_parity.py -q -m gpu -k "basis_change or GLT or chebyshev" > gpurun_out/s5/bchg_tests2.log 2>&1; echo "tests rc=$?"; tail -n 2 gpurun_out/s5/bchg_tests2.log
for rep in 1 2; do for cfg in "DG_BCHG=0" "DG_BCHG=1"; do echo -n "$cfg: " >> gpurun_out/s5/bchg_ab2.log; env $cfg python tools/bchg_ab.py >> gpurun_out/s5/bchg_ab2.log 2>&1; done; done
cat gpurun_out/s5/bchg_ab2.log
python bench.py > gpurun_out/s5/bench_c4_b.json 2> gpurun_out/s5/bench_c4_b.err; echo "bench rc=$?"
