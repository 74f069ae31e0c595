set -u
DG_K4_ALT=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/pytest_alt5.log 2>&1; echo "pytest alt rc=$?"
for v in 0 1 0 1; do DG_K4_ALT=$v python bench.py --steps 5 --warmup 3 --quick --degrees 4 > gpurun_out/bench_alt5_$v.json 2>/dev/null; grep -o '"p4": {[^}]*}' gpurun_out/bench_alt5_$v.json >> gpurun_out/alt5_ab.log; done; echo ab done
DG_K4_ALT=1 timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:k_kron4<\(int\)5, \(int\)2, \(int\)0" -s 2 -c 1 -o /tmp/prof_apply_n5a \
    python bench.py --steps 1 --warmup 0 --quick --degrees 4 > gpurun_out/ncu_apply_n5a.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/prof_apply_n5a.ncu-rep --page raw --csv > gpurun_out/apply_n5a_raw.csv 2>&1
ncu -i /tmp/prof_apply_n5a.ncu-rep --page source --csv --print-source sass > gpurun_out/apply_n5a_src.csv 2>&1
