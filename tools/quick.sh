#!/bin/bash
# quick GPU iteration: parity tests + condensed bench line
python -m pytest tests/test_parity_gpu.py -x -q 2>&1 | tail -2
python bench.py --steps ${STEPS:-20} --warmup 3 --no-cpu --no-loop ${BENCH_ARGS} 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('Mcol/s %.1f  ms/step %.4f  kernels %s  deep_frac %.3f  step_frac %.3f  e2e %s clocks %s' % (d['value']/1e6, d['ms_per_step'], {k: round(v,4) for k,v in d['kernels_ms'].items() if isinstance(v,float)}, d['roofline']['frac'], d['step_roofline']['frac'] or 0, d['e2e'] and round(d['e2e']['value']/1e6,1), d['clocks']))
"
