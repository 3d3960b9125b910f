# DRAM diagnostics for the two-level 25v kernel (pipe25, b_t = 2): where the excess over the algorithmic
# 60 B per update comes from, and whether TMA L2 eviction priorities move it.
#  * STENCIL_DBG=16: box B re-reads plane s (just loaded by box A) instead of plane q -- results are wrong,
#    the traffic difference is box B's 4-step re-read misses
#  * STENCIL_L2H=<a + 4b + 16c>: L2 priority of boxes A/B/C (1 evict_first, 2 evict_last, 3 normal)
M="--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -s 1 -c 1 --csv"
python tools/prof_case.py --workload C4 --T 4 > gpurun_out/dx_plain.log 2>&1 || exit 1
for w in C4 C5; do
  ncu $M -k regex:pipe25 python tools/prof_case.py --workload $w --T 4 > gpurun_out/dx_${w}_base.csv 2>&1
  STENCIL_DBG=16 ncu $M -k regex:pipe25 python tools/prof_case.py --workload $w --T 4 > gpurun_out/dx_${w}_b16.csv 2>&1
  for h in 2 6 16 32 26 42; do
    STENCIL_L2H=$h ncu $M -k regex:pipe25 python tools/prof_case.py --workload $w --T 4 > gpurun_out/dx_${w}_h$h.csv 2>&1
  done
done
for h in 0 2 6 16 26 42; do
  STENCIL_L2H=$h timeout 300 python bench.py --workload C4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary --alt-bt 0 > gpurun_out/dx_bench_C4_h$h.json 2>&1
done
# the 7v pipe kernel (C2, b_t = 4): box V (footprint) priority = a, box C (coefficients) = c
for h in 0 1 2 16 32 18 33; do
  STENCIL_L2H=$h ncu $M -k regex:pipe_kernel python tools/prof_case.py --workload C2 --bt 4 --T 8 > gpurun_out/dx_C2_h$h.csv 2>&1
done
for h in 0 2 18 33; do
  STENCIL_L2H=$h timeout 300 python bench.py --workload C2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary --alt-bt 0 > gpurun_out/dx_bench_C2_h$h.json 2>&1
done
