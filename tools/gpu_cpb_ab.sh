set -u
rm -f gpurun_out/ab.log
bash tools/gpu_r2_ab.sh "base n5c12 n5c20" 4
bash tools/gpu_r2_ab.sh "base n6c6 n6c10" 5
bash tools/gpu_r2_ab.sh "base n7c8 n7c12" 6
bash tools/gpu_r2_ab.sh "base n8c5" 7
bash tools/gpu_r2_ab.sh "base n9c4" 8
