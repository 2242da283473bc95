#!/bin/bash
# Launch list + ncu --set full captures of the kernels matching K (regex) for config CFG.
TAG=${TAG:-x}; CFG=${CFG:-2}; K=${K:-dec2_}
mkdir -p gpurun_out
CMD="python bench.py --config $CFG --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --only"
$CMD > gpurun_out/plain_${TAG}.log 2>&1 || { echo plain failed; tail gpurun_out/plain_${TAG}.log; exit 1; }
tail -1 gpurun_out/plain_${TAG}.log | cut -c1-300
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/launches_${TAG}.csv $CMD > /dev/null 2>&1
[ -n "$FULL" ] && ncu --set full --clock-control none --import-source on -k regex:$K -s ${SKIP:-2} -c ${COUNT:-2} \
    -o gpurun_out/prof_${TAG} $CMD > gpurun_out/ncu_${TAG}.log 2>&1
exit 0
