set -x
python bench.py --steps 3 --warmup 3 > gpurun_out/bench1.json 2> gpurun_out/bench1.err
echo "bench rc=$?"
python bench.py --steps 1 --warmup 1 --quick --degrees 2,5,8 > gpurun_out/plain_quick.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 1 --warmup 1 --quick --degrees 2,5,8 > gpurun_out/ncu_launch.log 2>&1
echo "ncu1 rc=$?"
python bench.py --steps 1 --warmup 0 --quick --degrees 5 > gpurun_out/plain_p5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_kron -s 46 -c 4 -o gpurun_out/prof_kron_p5 python bench.py --steps 1 --warmup 0 --quick --degrees 5 > gpurun_out/ncu_full.log 2>&1
echo "ncu2 rc=$?"
