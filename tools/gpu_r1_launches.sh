set -u
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_full.csv python bench.py --steps 2 --warmup 1 --quick > gpurun_out/launches_full.log 2>&1; echo "launches rc=$?"
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --workload c2 > gpurun_out/bench_c2_chunk4.json 2>/dev/null; echo "c2 rc=$?"
