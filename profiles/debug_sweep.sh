#!/bin/bash
# Timing experiment: skeleton cost of the pipeline (POLY_DEBUG bits: 1 skip
# compute, 2 skip look-back).  Outputs are wrong under POLY_DEBUG != 0.
TAG=${TAG:-dbg}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_${TAG}.log 2>&1
for C in ${CONFIGS:-2}; do
  for D in ${DFLAGS:-0 1 2 3}; do
    POLY_DEBUG=$D timeout 300 python bench.py --config $C --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-roundtrip-check \
      > gpurun_out/dbg_${TAG}_cfg${C}_d$D.json 2> gpurun_out/dbg_${TAG}_cfg${C}_d$D.err
  done
done
