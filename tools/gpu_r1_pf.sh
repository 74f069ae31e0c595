for pf in 0 1 2; do
DG_L2PF=$pf timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --degrees 3,5,7 > gpurun_out/bench_pf$pf.json 2> gpurun_out/bench_pf$pf.err
DG_L2PF=$pf timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k 'regex:k_kron4<\(int\)6' -c 12 --csv python bench.py --steps 1 --warmup 0 --quick --degrees 5 > gpurun_out/ncu_pf$pf.csv 2>&1
done
DG_L2PF=0 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --workload c3 > gpurun_out/bench_q3pf0.json 2> gpurun_out/bench_q3pf0.err
echo done
