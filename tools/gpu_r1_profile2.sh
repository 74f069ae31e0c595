set -x
python -m pytest tests/test_gpu_parity.py -x -q -k "apply or access or gl_basis or chebyshev or c2" > gpurun_out/pytest2.log 2>&1
echo "pytest rc=$?"
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench2.json 2> gpurun_out/bench2.err
echo "bench rc=$?"
python bench.py --steps 1 --warmup 0 --quick --degrees 5 > gpurun_out/plain_p5b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_kron -s 15 -c 2 -o gpurun_out/prof_kron_p5 python bench.py --steps 1 --warmup 0 --quick --degrees 5 > gpurun_out/ncu_full2.log 2>&1
echo "ncu rc=$?"
