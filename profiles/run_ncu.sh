#!/bin/bash
# Profiling recipe used for profiles/ (run on the B200 box via gpurun).
# For each config in CONFIGS: 1) plain run, 2) launch list of our kernels,
# 3) one `ncu --set full` capture per kernel regex in KERNELS.
TAG=${TAG:-r01}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_${TAG}.log 2>&1
for CFG in ${CONFIGS:-2}; do
  CMD="python bench.py --config $CFG --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
  $CMD > gpurun_out/plain_${TAG}_cfg${CFG}.log 2>&1 || { echo "plain run failed cfg$CFG"; continue; }
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:poly_ \
      --csv --log-file gpurun_out/launches_${TAG}_cfg${CFG}.csv $CMD > gpurun_out/ncu_launch_${TAG}_cfg${CFG}.log 2>&1
  for K in ${KERNELS:-poly_compress poly_decompress}; do
    ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 \
        -o gpurun_out/prof_${TAG}_cfg${CFG}_$K $CMD > gpurun_out/ncu_full_${TAG}_cfg${CFG}_$K.log 2>&1 || true
  done
done
exit 0
