#!/bin/bash
# One gpurun call: GPU tests, the default bench line, the ncu launch list of
# the headline command per config and one ncu --set full capture per kernel,
# exported to small text summaries (the .ncu-rep files are deleted unless
# KEEP_REP=1: gpurun copies back at most 64 MiB).
# usage: TAG=r03c NCU_CFGS="5 2" bash profiles/session_measure.sh
TAG=${TAG:-r03}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_${TAG}.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_throttle_reasons.active --format=csv > gpurun_out/gpu_${TAG}.txt 2>&1
if [ -z "$NOTEST" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_${TAG}.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest_${TAG}.log
fi
if [ -z "$NOBENCH" ]; then
  timeout 900 python bench.py > gpurun_out/bench_${TAG}_default.json 2> gpurun_out/bench_${TAG}_default.err
fi
CMD="python bench.py --only --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-roundtrip-check"
for CFG in ${NCU_CFGS:-5}; do
  C="$CMD --config $CFG"
  if timeout 300 $C > gpurun_out/plain_${TAG}_cfg$CFG.log 2>&1; then
    timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
        --csv --log-file gpurun_out/launches_${TAG}_cfg$CFG.csv $C > gpurun_out/ncu_launch_${TAG}_cfg$CFG.log 2>&1
    case $CFG in 2|6) KS=${KERNELS:-poly_compress_pipe poly_decompress_pipe dec3_main};; 3) KS="poly_compress_large poly_decompress_large";; *) KS=${KERNELS:-cmp3 dec3_main};; esac
    for K in $KS; do
      R=gpurun_out/full_${TAG}_cfg${CFG}_$K
      timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 -o $R $C > $R.log 2>&1
      if [ -f $R.ncu-rep ]; then
        python profiles/ncu_summary.py $R.ncu-rep > $R.summary.txt 2>&1
        python profiles/src_lines.py $R.ncu-rep 40 > $R.src_lines.txt 2>&1
        python profiles/stall_lines.py $R.ncu-rep 40 > $R.stall_lines.txt 2>&1
        [ -z "$KEEP_REP" ] && rm -f $R.ncu-rep
      fi
    done
  fi
done
du -sh gpurun_out
exit 0
