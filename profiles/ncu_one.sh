#!/bin/bash
# One ncu --set full capture of kernel regex K for bench config CFG, with
# optional POLY_DEBUG timing flags (outputs wrong when nonzero).
TAG=${TAG:-x}; CFG=${CFG:-2}; K=${K:-poly_decompress_pipe}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_${TAG}.log 2>&1
CMD="python bench.py --config $CFG --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-roundtrip-check"
$CMD > gpurun_out/plain_${TAG}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 -o gpurun_out/prof_${TAG} $CMD > gpurun_out/ncu_${TAG}.log 2>&1
exit 0
