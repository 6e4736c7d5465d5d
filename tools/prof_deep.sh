#!/bin/bash
# ncu --set full of the deep + shallow kernels of a short bench run (1 GPU)
TAG=${1:-prof}
python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-deep_kernel|shallow_kernel}" -s 3 -c ${COUNT:-2} -o gpurun_out/${TAG} python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/${TAG}_ncu.log 2>&1
tail -2 gpurun_out/${TAG}_ncu.log
