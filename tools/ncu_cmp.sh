M=gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none -k regex:"deep_tpc|shallow_kernel|redo|fix" -c 4 python tools/steptime.py --steps 2 --reps 1 ser:CVG_OVERLAP=0 > gpurun_out/ncu_new.txt 2>&1
CONVGPU_LIB=tools/libconvgpu_head.so ncu --metrics $M --clock-control none -k regex:"deep_tpc|shallow_kernel" -c 2 python tools/steptime.py --steps 2 --reps 1 ser:CVG_OVERLAP=0 > gpurun_out/ncu_head.txt 2>&1
python tools/steptime.py --kernels base guard0:CVG_GUARD=0 ser:CVG_OVERLAP=0 ser_g0:CVG_OVERLAP=0,CVG_GUARD=0 > gpurun_out/st_new.txt 2>&1
for f in gpurun_out/ncu_new.txt gpurun_out/ncu_head.txt; do echo $f; grep -E "^  [a-z]|duration|inst_exec|dram" $f; done; cat gpurun_out/st_new.txt
