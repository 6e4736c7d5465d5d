#!/bin/bash
# One GPU iteration: parity tests, the default bench line, the kernels alone.
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
bash tools/quick.sh 2>&1 | tail -1
j() { python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['kernels_ms'].items() if isinstance(v,float)})"; }
CVG_OVERLAP=0 python bench.py --steps 20 --warmup 3 --no-cpu --no-loop --no-e2e | j nooverlap
for v in $EXTRA; do env $v python bench.py --steps 20 --warmup 3 --no-cpu --no-loop --no-e2e | j "$v"; done
