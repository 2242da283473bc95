#!/bin/bash
# Profiling recipe used for profiles/ (run on the B200 box via gpurun).
# 1) plain run, 2) launch list of our kernels, 3) one full capture per top kernel.
set -e
CFG=${CFG:-2}
TAG=${TAG:-r01}
CMD="python bench.py --config $CFG --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
mkdir -p gpurun_out
$CMD > gpurun_out/plain_${TAG}_cfg${CFG}.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:poly_ \
    --csv --log-file gpurun_out/launches_${TAG}_cfg${CFG}.csv $CMD > gpurun_out/ncu_launch_${TAG}_cfg${CFG}.log 2>&1
for K in ${KERNELS:-poly_compress_tiled poly_decompress_tiled}; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 \
      -o gpurun_out/prof_${TAG}_cfg${CFG}_$K $CMD > gpurun_out/ncu_full_${TAG}_cfg${CFG}_$K.log 2>&1 || true
done
