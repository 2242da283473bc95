#!/bin/bash
# A/B timing of library variants: VARIANTS="name=path ..." (path relative to the repo root).
TAG=${TAG:-ab}
mkdir -p gpurun_out
for V in $VARIANTS; do
  NAME=${V%%=*}; LIB=${V#*=}
  if [ -n "$TESTS" ]; then
    POLY_LIB=$PWD/$LIB timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_${TAG}_$NAME.log 2>&1; echo "exit $?" >> gpurun_out/pytest_${TAG}_$NAME.log
  fi
  for C in ${CONFIGS:-2}; do
    POLY_LIB=$PWD/$LIB timeout 120 python bench.py --config $C --steps 10 --warmup 3 --no-e2e --no-cpu-baseline \
      > gpurun_out/ab_${TAG}_${NAME}_cfg$C.json 2> gpurun_out/ab_${TAG}_${NAME}_cfg$C.err
  done
done
