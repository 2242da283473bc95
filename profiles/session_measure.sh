#!/bin/bash
# One gpurun call: GPU tests, the default bench line, per-config quick lines,
# the ncu launch list of the headline command and ncu --set full captures of
# the headline config's kernels.  usage: TAG=r03a bash profiles/session_measure.sh
TAG=${TAG:-r03}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_${TAG}.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_throttle_reasons.active --format=csv > gpurun_out/gpu_${TAG}.txt 2>&1
if [ -z "$NOTEST" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_${TAG}.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest_${TAG}.log
fi
timeout 900 python bench.py > gpurun_out/bench_${TAG}_default.json 2> gpurun_out/bench_${TAG}_default.err
CMD="python bench.py --only --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-roundtrip-check"
for CFG in ${NCU_CFGS:-5}; do
  C="$CMD --config $CFG"
  if timeout 300 $C > gpurun_out/plain_${TAG}_cfg$CFG.log 2>&1; then
    timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
        --csv --log-file gpurun_out/launches_${TAG}_cfg$CFG.csv $C > gpurun_out/ncu_launch_${TAG}_cfg$CFG.log 2>&1
    for K in ${KERNELS:-poly_compress dec3_main}; do
      timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 \
          -o gpurun_out/full_${TAG}_cfg${CFG}_$K $C > gpurun_out/ncu_full_${TAG}_cfg${CFG}_$K.log 2>&1
    done
  fi
done
exit 0
