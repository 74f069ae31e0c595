# Fresh ncu --set full captures of the weakest kernels on the current code (round 2, session 3):
# the odd-n Chebyshev steps (n = 3, 7), the n = 6 Chebyshev step, and k_quad3 on C3.
set -u
mkdir -p gpurun_out/pf /tmp/pf
bash tools/ncu_capture.sh pf/cheby_p2 k_kron4 2 1 python tools/prof_driver.py 2 cheby 2
bash tools/ncu_capture.sh pf/cheby_p6 k_kron4 2 1 python tools/prof_driver.py 6 cheby 2
bash tools/ncu_capture.sh pf/cheby_p5 k_kron4 2 1 python tools/prof_driver.py 5 cheby 2
bash tools/ncu_capture.sh pf/quad3_c3 k_quad3 1 1 python tools/prof_driver.py C3 apply 2
for n in cheby_p2 cheby_p6 cheby_p5 quad3_c3; do
  zcat gpurun_out/pf/${n}_src.csv.gz > /tmp/${n}_src.csv
  python tools/ncu_segments.py /tmp/${n}_src.csv > gpurun_out/pf/${n}_segments.txt 2>&1
  python tools/ncu_sass_mix.py /tmp/${n}_src.csv $(python -c "from synthetic import CONFIGS, c4_spec; n=\"$n\".split(\"_\")[1]; print((CONFIGS[n.upper()] if n.upper() in CONFIGS else c4_spec(int(n[1:]))).n_dofs)") > gpurun_out/pf/${n}_mix.txt 2>&1
done
ls -la gpurun_out/pf
