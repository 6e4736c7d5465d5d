#!/bin/bash
# A/B step timings on one GPU: each argument is "label|ENV=... ENV2=..." ;
# prints ms/step and the deep kernel's time per configuration.
for spec in "$@"; do
  label=${spec%%|*}; envs=${spec#*|}
  env $envs python bench.py --steps ${STEPS:-30} --warmup 5 --no-cpu --no-loop --no-e2e ${BENCH_ARGS} 2>"gpurun_out/ab_${label//\//_}.err" | tail -1 | \
  python -c "
import json,sys
d=json.loads(sys.stdin.read())
k=d['kernels_ms']
print('%-28s step %.4f ms  deep %.4f  trig %.4f  sh_tail %.4f' % ('$label', d['ms_per_step'], k['deep'], k['trigger_groups'], k['shallow_tail_after_deep']))
"
done
