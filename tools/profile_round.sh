#!/bin/bash
# Round profiling recipe (B200_PROFILING.md): plain bench run, then the
# launch list of the same command, then one --set full capture of the top
# kernels.  Outputs under gpurun_out/<tag>_*; summaries are copied to
# profiles/ by tools/summarize_profile.py.
TAG=${1:-r01}
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-loop"
$CMD > gpurun_out/${TAG}_plain.json 2> gpurun_out/${TAG}_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_launches.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"deep_|shallow_kernel|shallow_tile_kernel|trigger_groups|redo_kernel" -s 12 -c 4 -o gpurun_out/${TAG}_full $CMD > gpurun_out/${TAG}_full.log 2>&1
echo "rc=$?"
tail -2 gpurun_out/${TAG}_full.log
