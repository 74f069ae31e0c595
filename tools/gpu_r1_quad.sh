set -x
python bench.py --steps 1 --warmup 0 --quick --workload c3 > gpurun_out/plain_c3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_quad -s 15 -c 2 -o gpurun_out/prof_quad_c3 python bench.py --steps 1 --warmup 0 --quick --workload c3 > gpurun_out/ncu_quad.log 2>&1
echo "ncu rc=$?"
