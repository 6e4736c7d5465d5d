#!/bin/bash
# Load-imbalance stress (BASELINE config 5): per-rank step time of each
# share of a W-way partition (bench.py --slice), balanced vs naive.
# Prints config, partition, W, max and min over ranks (ms).
for cfg in ${CFGS:-c5_05 c5_50 c5_95 c4}; do
  for part in balanced naive; do
    for W in ${WAYS:-8}; do
      ts=""
      for r in $(seq 0 $((W - 1))); do
        t=$(python bench.py --config $cfg --partition $part --slice $r/$W --steps 20 --warmup 3 --no-cpu --no-loop --no-e2e 2>/dev/null \
            | python -c "import json,sys; print(json.loads(sys.stdin.read())['ms_per_step'])")
        ts="$ts $t"
      done
      python -c "import sys; v=[float(x) for x in sys.argv[4:]]; print(sys.argv[1], sys.argv[2], sys.argv[3], 'max %.4f min %.4f ms' % (max(v), min(v)))" $cfg $part $W $ts
    done
  done
done
