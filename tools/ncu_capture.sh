# ncu --set full of one kernel launch, exported to CSV on the box (raw + source pages) and
# summarised; the .ncu-rep is deleted so gpurun_out stays small.
# usage: tools/ncu_capture.sh NAME KERNEL_REGEX SKIP COUNT cmd...
set -u
name=$1; kre=$2; skip=$3; cnt=$4; shift 4
"$@" > gpurun_out/${name}_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:$kre -s $skip -c $cnt -o /tmp/${name} "$@" > gpurun_out/${name}_ncu.log 2>&1
ncu -i /tmp/${name}.ncu-rep --page raw --csv > gpurun_out/${name}_raw.csv 2>/dev/null
ncu -i /tmp/${name}.ncu-rep --page source --csv > /tmp/${name}_src.csv 2>/dev/null
gzip -c /tmp/${name}_src.csv > gpurun_out/${name}_src.csv.gz
python tools/ncu_summary_csv.py gpurun_out/${name}_raw.csv > gpurun_out/${name}_summary.txt 2>&1
ls -la gpurun_out/${name}_*
