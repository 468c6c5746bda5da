# Bench lines for every config plus one-step ncu launch lists (c2, c5) into gpurun_out/r/.
# Usage (GPU box): bash tools/refresh_profiles.sh
set -x
mkdir -p gpurun_out/r
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/r/c2.json 2> gpurun_out/r/c2.err
for c in c2_concat c1 c5_inner c4; do timeout 400 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/r/$c.json 2> gpurun_out/r/$c.err; done
timeout 300 python tools/one_step.py c2_inner 256 > /dev/null 2>&1 && \
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r/c2_launches.csv python tools/one_step.py c2_inner 256 > gpurun_out/r/ncu_c2.log 2>&1
timeout 300 python tools/one_step.py c5_inner 256 > /dev/null 2>&1 && \
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r/c5_launches.csv python tools/one_step.py c5_inner 256 > gpurun_out/r/ncu_c5.log 2>&1
ls -la gpurun_out/r
