# Round 2 session 5 evidence (k_bchgw as the basis-change default at n = 3, 5, 6, 7, 9):
# launch list and shares, DRAM traffic per launch (k_kron* and k_bchg*), ncu --set full of
# k_bchgw at p = 4 and p = 6 (n = 5, 7) and of the block-staged k_bchg at p = 4 for comparison.
set -u
mkdir -p gpurun_out/s5 /tmp/s5
python bench.py --steps 2 --warmup 1 --quick > gpurun_out/s5/quick_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/s5/launches.csv \
    python bench.py --steps 2 --warmup 1 --quick > gpurun_out/s5/launches.log 2>&1; echo "launches rc=$?"
python tools/launch_share.py gpurun_out/s5/launches.csv > gpurun_out/s5/launch_share.txt 2>&1
python bench.py --steps 1 --warmup 0 --quick > gpurun_out/s5/traffic_plain.json 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --kernel-name-base demangled \
    -k regex:"k_kron|k_bchg" --csv python bench.py --steps 1 --warmup 0 --quick > gpurun_out/s5/traffic_ncu.csv 2> gpurun_out/s5/traffic.err; echo "traffic rc=$?"
python tools/traffic_from_ncu.py gpurun_out/s5/traffic_ncu.csv gpurun_out/s5/r2s5_traffic.json gpurun_out/s5/r2s5_traffic_ncu.csv
bash tools/ncu_capture.sh s5/bchgw_p4 k_bchg[wp] 1 1 python tools/prof_driver.py 4 bchg 2
bash tools/ncu_capture.sh s5/bchgw_p6 k_bchg[wp] 1 1 python tools/prof_driver.py 6 bchg 2
DG_BCHG=1 bash tools/ncu_capture.sh s5/bchg_p4 k_bchg\< 1 1 python tools/prof_driver.py 4 bchg 2
for n in bchgw_p4 bchgw_p6 bchg_p4; do
  zcat gpurun_out/s5/${n}_src.csv.gz > /tmp/${n}_src.csv
  p=$(echo $n | sed 's/.*_p//'); nd=$(python -c "from synthetic import c4_spec; print(c4_spec($p).n_dofs)")
  python tools/ncu_sass_mix.py /tmp/${n}_src.csv $nd > gpurun_out/s5/${n}_mix.txt 2>&1
done
ls -la gpurun_out/s5
