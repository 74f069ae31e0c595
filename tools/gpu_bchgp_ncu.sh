set -u
mkdir -p gpurun_out/bpn /tmp/bpn
export DG_BCHG=5 DG_BCHGW_MODE=4
for p in 3 5 6; do
  bash tools/ncu_capture.sh bpn/bchgp_p$p k_bchgp 1 1 python tools/prof_driver.py $p bchg 2 > /dev/null 2>&1
  nd=$(python -c "from synthetic import c4_spec; print(c4_spec($p).n_dofs)")
  python tools/ncu_sass_mix.py /tmp/bpn/bchgp_p${p}_src.csv $nd > gpurun_out/bpn/bchgp_p${p}_mix.txt 2>&1
  rm -f gpurun_out/bpn/bchgp_p${p}_src.csv.gz
  grep -E "duration|dram__bytes|lsu_wavefronts|bank_conflicts|warps_active|registers|occupancy_limit|fp64|issue_active|stalled|hit_rate|shared_mem_per_block" gpurun_out/bpn/bchgp_p${p}_summary.txt
  head -25 gpurun_out/bpn/bchgp_p${p}_mix.txt
done
