# One training step's launch list with time, DRAM bytes, tensor-pipe % and issue % per kernel
# (ncu, cold-cache and serialised: compare shares).  Usage (GPU box):
#   bash tools/step_metrics.sh <config> <B> <out.csv>
set -e
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active
timeout 300 python tools/one_step.py "$1" "$2" > /dev/null
timeout 1200 ncu --profile-from-start off --metrics $M --clock-control none --print-units base --csv --log-file "$3" \
  python tools/one_step.py "$1" "$2" > /dev/null
