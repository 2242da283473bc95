#!/bin/bash
# Round-end measurement in one gpurun call: default bench line (cfg2 with e2e
# and the CPU oracle baseline), the other configs, the ncu launch list of the
# default command and one `ncu --set full` capture per pipeline kernel.
# usage: TAG=r02 bash profiles/round_measure.sh
TAG=${TAG:-r02}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_${TAG}.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_throttle_reasons.active --format=csv > gpurun_out/gpu_${TAG}.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench_${TAG}_default.json 2> gpurun_out/bench_${TAG}_default.err
for C in ${CONFIGS:-1 3 4 5}; do
  timeout 300 python bench.py --config $C --steps 10 --warmup 3 > gpurun_out/bench_${TAG}_cfg$C.json 2> gpurun_out/bench_${TAG}_cfg$C.err
done
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-roundtrip-check"
if $CMD > gpurun_out/plain_${TAG}.log 2>&1; then
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:poly_ \
      --csv --log-file gpurun_out/launches_${TAG}_cfg2.csv $CMD > gpurun_out/ncu_launch_${TAG}.log 2>&1
  for K in poly_compress_pipe poly_decompress_pipe; do
    ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 -o gpurun_out/full_${TAG}_cfg2_$K $CMD \
        > gpurun_out/ncu_full_${TAG}_$K.log 2>&1
  done
fi
exit 0
