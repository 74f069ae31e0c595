# Round-2 final evidence on one B200: the NCCL multi-rank worker at world size 1 (script check; the
# >= 2-GPU test skips here), bench line, reference arm, k_kron3c ncu capture, traffic of k_kron3c.
set -u
mkdir -p gpurun_out/fin /tmp/fin
python -m torch.distributed.run --nnodes=1 --nproc-per-node=1 --master-addr 127.0.0.1 --master-port 29533 tests/_nccl_ranks.py > gpurun_out/fin/nccl_worker_w1.log 2>&1; echo "worker rc=$?"; tail -2 gpurun_out/fin/nccl_worker_w1.log
python -m pytest tests/test_gpu_nccl_multirank.py -q -m gpu > gpurun_out/fin/nccl_test.log 2>&1; tail -1 gpurun_out/fin/nccl_test.log
python bench.py > gpurun_out/fin/bench_c4.json 2> gpurun_out/fin/bench_c4.err; echo "bench rc=$?"
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/fin/bench_reference.json 2> gpurun_out/fin/bench_reference.err; echo "ref rc=$?"
python bench.py --steps 1 --warmup 0 --quick --degrees 2 > gpurun_out/fin/traffic_plain.json 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --kernel-name-base demangled \
    -k regex:k_kron --csv python bench.py --steps 1 --warmup 0 --quick --degrees 2 > gpurun_out/fin/traffic_ncu_p2.csv 2> gpurun_out/fin/traffic.err; echo "traffic rc=$?"
bash tools/ncu_capture.sh fin/k3c_cheby_p2 k_kron3c 2 1 python tools/prof_driver.py 2 cheby 2
bash tools/ncu_capture.sh fin/k3c_apply_p2 k_kron3c 1 1 python tools/prof_driver.py 2 apply 2
for n in k3c_cheby_p2 k3c_apply_p2; do
  zcat gpurun_out/fin/${n}_src.csv.gz > /tmp/${n}_src.csv
  python tools/ncu_segments.py /tmp/${n}_src.csv > gpurun_out/fin/${n}_segments.txt 2>&1
  python tools/ncu_sass_mix.py /tmp/${n}_src.csv 110592000 > gpurun_out/fin/${n}_mix.txt 2>&1
done
ls -la gpurun_out/fin
