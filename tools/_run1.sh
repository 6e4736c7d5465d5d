echo "== alone (thr 2.0)"; python tools/steptime.py --thr 2.0 --steps 50 --reps 3 "old:CVG_SHALLOW_TILE=0" "tile8" "tile9:CVG_TILE_WARPS=9" 2>&1 | tail -3
for t in ch3 ch4; do CONVGPU_LIB=$PWD/tools/libconvgpu_$t.so python tools/steptime.py --thr 2.0 --steps 50 --reps 3 "tile8_$t" 2>&1 | tail -1; done
echo "== overlapped"; python tools/steptime.py --steps 50 --reps 3 --kernels "old:CVG_SHALLOW_TILE=0" "tile24" 2>&1 | tail -2
for t in ch3 ch4; do CONVGPU_LIB=$PWD/tools/libconvgpu_$t.so python tools/steptime.py --steps 50 --reps 3 --kernels "tile24_$t" 2>&1 | tail -1; done
for t in nw20 nw22 nw23; do CONVGPU_LIB=$PWD/tools/libconvgpu_$t.so python tools/steptime.py --steps 50 --reps 3 --kernels "tile8_$t" "tile9_$t:CVG_TILE_WARPS=9" "tile7_$t:CVG_TILE_WARPS=7" 2>&1 | tail -3; done
