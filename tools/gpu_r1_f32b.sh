timeout 600 python tools/f32_errors.py > gpurun_out/f32_errors.txt 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_f32.json 2> gpurun_out/bench_f32.err
echo done
