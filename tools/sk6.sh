B="python bench.py --workload C4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary --alt-bt 0"
STENCIL_XG=4 STENCIL_DBG=64 timeout 300 $B --tile-cfg 3 > gpurun_out/sk6_nowait.json 2>&1
STENCIL_XG=4 STENCIL_DBG=192 timeout 300 $B --tile-cfg 3 > gpurun_out/sk6_nowait_nofence.json 2>&1
STENCIL_XG=4 STENCIL_DBG=128 timeout 300 $B --tile-cfg 3 > gpurun_out/sk6_nofence.json 2>&1
STENCIL_XG=4 STENCIL_SCHED=0 timeout 300 $B --tile-cfg 3 > gpurun_out/sk6_dyn.json 2>&1
