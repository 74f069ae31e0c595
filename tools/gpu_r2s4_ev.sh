# Round 2 session 4 evidence for the transformed-residual Chebyshev step (KMODE_CHEBY_GLT):
# variant parity, bench line, launch list, DRAM traffic per launch, ncu --set full of the GLT
# step at p = 4, 7 (n = 5, 8) and of the direct step at p = 4 (non-first steps: skip 3).
set -u
mkdir -p gpurun_out/s4 /tmp/s4
python -m pytest tests/test_gpu_variants.py -q -m gpu -k "GLT" > gpurun_out/s4/variants.log 2>&1; echo "variants rc=$?"; tail -1 gpurun_out/s4/variants.log
python bench.py > gpurun_out/s4/bench_c4.json 2> gpurun_out/s4/bench_c4.err; echo "bench rc=$?"
python bench.py --steps 2 --warmup 1 --quick > gpurun_out/s4/quick_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/s4/launches.csv \
    python bench.py --steps 2 --warmup 1 --quick > gpurun_out/s4/launches.log 2>&1; echo "launches rc=$?"
python tools/launch_share.py gpurun_out/s4/launches.csv > gpurun_out/s4/launch_share.txt 2>&1
python bench.py --steps 1 --warmup 0 --quick > gpurun_out/s4/traffic_plain.json 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --kernel-name-base demangled \
    -k regex:k_kron --csv python bench.py --steps 1 --warmup 0 --quick > gpurun_out/s4/traffic_ncu.csv 2> gpurun_out/s4/traffic.err; echo "traffic rc=$?"
python tools/traffic_from_ncu.py gpurun_out/s4/traffic_ncu.csv gpurun_out/s4/r2s4_traffic.json profiles/r2s4_traffic_ncu.csv
bash tools/ncu_capture.sh s4/glt_cheby_p4 k_kron4 3 1 python tools/prof_driver.py 4 cheby 2
bash tools/ncu_capture.sh s4/glt_cheby_p7 k_kron4 3 1 python tools/prof_driver.py 7 cheby 2
DG_CHEBY_GLT=0 bash tools/ncu_capture.sh s4/gl_cheby_p4 k_kron4 3 1 python tools/prof_driver.py 4 cheby 2
for n in glt_cheby_p4 glt_cheby_p7 gl_cheby_p4; do
  zcat gpurun_out/s4/${n}_src.csv.gz > /tmp/${n}_src.csv
  python tools/ncu_segments.py /tmp/${n}_src.csv > gpurun_out/s4/${n}_segments.txt 2>&1
  p=$(echo $n | sed 's/.*_p//'); nd=$(python -c "from synthetic import c4_spec; print(c4_spec($p).n_dofs)")
  python tools/ncu_sass_mix.py /tmp/${n}_src.csv $nd > gpurun_out/s4/${n}_mix.txt 2>&1
done
ls -la gpurun_out/s4
