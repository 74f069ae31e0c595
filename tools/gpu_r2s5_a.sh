# Round 2 session 5, step A: parity of the new basis-change defaults, standalone A/B, the GLT mask
# re-check at n = 6 with the faster b~ pass, then the default bench line.
set -u
mkdir -p gpurun_out/s5
python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py tests/test_gpu_mixed_precision.py -q -m gpu -k "basis_change" > gpurun_out/s5/bchg_tests.log 2>&1; echo "bchg tests rc=$?"; tail -n 2 gpurun_out/s5/bchg_tests.log
for rep in 1 2; do for cfg in "DG_BCHG=0" "DG_BCHG=1"; do echo -n "$cfg: " >> gpurun_out/s5/bchg_ab.log; env $cfg python tools/bchg_ab.py >> gpurun_out/s5/bchg_ab.log 2>&1; done; done
cat gpurun_out/s5/bchg_ab.log
bash tools/gpu_env_ab.sh "DG_CHEBY_GLT=119 DG_CHEBY_GLT=127 DG_BCHG=1" 4,5,6; cat gpurun_out/envab.log
python bench.py > gpurun_out/s5/bench_c4.json 2> gpurun_out/s5/bench_c4.err; echo "bench rc=$?"
