timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_quad3 -s 1 -c 1 -o gpurun_out/prof_q3 python bench.py --steps 1 --warmup 0 --quick --workload c3 > gpurun_out/ncu_q3.log 2>&1
echo "ncu rc=$?"
ls -la gpurun_out/prof_q3.ncu-rep
