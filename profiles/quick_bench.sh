#!/bin/bash
# compress / decompress GB/s of each config in CFGS (short runs, no e2e / CPU baseline)
for c in ${CFGS:-2 4 5 3}; do
  python bench.py --config $c --steps ${STEPS:-3} --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/qb_$c.json 2> gpurun_out/qb_$c.err || { echo "cfg$c failed"; tail -2 gpurun_out/qb_$c.err; continue; }
  python -c "import json,sys; d=json.load(open('gpurun_out/qb_$c.json')); print('cfg$c', d['config']['workload'], 'C', d['compress_gbs'], 'D', d['decompress_gbs'], 'frac', d['roofline']['frac'])"
done
