#!/bin/bash
# One gpurun call: GPU parity tests, a plain bench line per config, the ncu
# launch list of the default bench command.  Usage: TAG=r01b bash profiles/gpu_check.sh
TAG=${TAG:-r01}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_${TAG}.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_${TAG}.log 2>&1
timeout ${PYTEST_TIMEOUT:-420} python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu_${TAG}.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_${TAG}.log
for C in ${CONFIGS:-2 1 3 4 5}; do
  timeout 180 python bench.py --config $C --steps 10 --warmup 3 ${BENCH_ARGS} > gpurun_out/bench_${TAG}_cfg$C.json 2> gpurun_out/bench_${TAG}_cfg$C.err
done
if [ -n "$NCU" ]; then
  CMD="python bench.py --config 2 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
  $CMD > gpurun_out/plain_${TAG}.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:poly_ \
      --csv --log-file gpurun_out/launches_${TAG}_cfg2.csv $CMD > gpurun_out/ncu_launch_${TAG}.log 2>&1
fi
exit 0
