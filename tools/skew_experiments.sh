# The experiments behind DESIGN.md §5d (skewed 25v tiles, tile_cfg 3) and the cluster-pair stall
# attribution, in the order they were run (gpurun calls sk2, sk6, sk7, sk8, pp).  Every STENCIL_DBG bit
# used here gives wrong results on purpose: they remove parts of the synchronisation to measure their cost.
#   bash tools/skew_experiments.sh [mismatch|sync|ncu|ceiling|pair|all]
# (tools/skew_check.sh: the tests + sustained rates + ncu of the plan itself)
what=${1:-all}
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary --alt-bt 0"
FULL="ncu --set full --clock-control none --import-source on -k regex:pipe25 -s 1 -c 1"
if [ "$what" = mismatch ] || [ "$what" = all ]; then  # where a wrong plan differs from the naive sweeps
  python tools/dbg_skew.py 130 37 41 2 > gpurun_out/sk2_a.log 2>&1        # default z-chunks
  python tools/dbg_skew.py 130 37 41 2 1000 > gpurun_out/sk2_e.log 2>&1   # one z-chunk
  python tools/dbg_skew.py 24 60 20 2 > gpurun_out/sk2_c.log 2>&1
fi
if [ "$what" = sync ] || [ "$what" = all ]; then  # sustained C4 without the wait / the fence / both
  STENCIL_XG=4 STENCIL_DBG=64 timeout 300 $B --workload C4 --tile-cfg 3 > gpurun_out/sk6_nowait.json 2>&1
  STENCIL_XG=4 STENCIL_DBG=192 timeout 300 $B --workload C4 --tile-cfg 3 > gpurun_out/sk6_nowait_nofence.json 2>&1
  STENCIL_XG=4 STENCIL_DBG=128 timeout 300 $B --workload C4 --tile-cfg 3 > gpurun_out/sk6_nofence.json 2>&1
  STENCIL_XG=4 STENCIL_SCHED=0 timeout 300 $B --workload C4 --tile-cfg 3 > gpurun_out/sk6_dyn.json 2>&1
fi
if [ "$what" = ncu ] || [ "$what" = all ]; then  # stall attribution: skewed without wait/fence vs the default
  python tools/prof_case.py --workload C4 --T 4 --cfg 3 > gpurun_out/sk7_plain.log 2>&1 || exit 1
  STENCIL_DBG=192 timeout 600 $FULL -o gpurun_out/sk7_c4_cfg3_nowait python tools/prof_case.py --workload C4 --T 4 --cfg 3 > gpurun_out/sk7_ncu1.log 2>&1
  timeout 600 $FULL -o gpurun_out/sk7_c4_cfg0 python tools/prof_case.py --workload C4 --T 4 --cfg 0 > gpurun_out/sk7_ncu2.log 2>&1
fi
if [ "$what" = ceiling ] || [ "$what" = all ]; then  # compute only: no wait, no fence, no release store
  M="--metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -s 1 -c 1 --csv"
  STENCIL_DBG=448 timeout 600 ncu $M -k regex:pipe25 python tools/prof_case.py --workload C4 --T 4 --cfg 3 > gpurun_out/sk8_ncu_c4_compute.csv 2>&1
  STENCIL_DBG=448 timeout 600 ncu $M -k regex:pipe25 python tools/prof_case.py --workload C5 --T 4 --cfg 3 > gpurun_out/sk8_ncu_c5_compute.csv 2>&1
  STENCIL_DBG=448 timeout 300 $B --workload C4 --tile-cfg 3 > gpurun_out/sk8_bench_c4.json 2>&1
  STENCIL_DBG=448 timeout 300 $B --workload C5 --tile-cfg 3 > gpurun_out/sk8_bench_c5.json 2>&1
fi
if [ "$what" = pair ] || [ "$what" = all ]; then  # cluster-pair tiles (tile_cfg 1): stall attribution
  python tools/prof_case.py --workload C4 --T 4 --cfg 1 > gpurun_out/pp_plain.log 2>&1 || exit 1
  timeout 600 $FULL -o gpurun_out/pp_c4_cfg1 python tools/prof_case.py --workload C4 --T 4 --cfg 1 > gpurun_out/pp_ncu.log 2>&1
fi
