# skewed tiles, compute only (STENCIL_DBG=448: no flag wait, no fence, no release store; wrong results)
python tools/prof_case.py --workload C4 --T 4 --cfg 3 > gpurun_out/sk8_plain.log 2>&1 || exit 1
M="--metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -s 1 -c 1 --csv"
STENCIL_DBG=448 timeout 600 ncu $M -k regex:pipe25 python tools/prof_case.py --workload C4 --T 4 --cfg 3 > gpurun_out/sk8_ncu_c4_compute.csv 2>&1
STENCIL_DBG=448 timeout 600 ncu $M -k regex:pipe25 python tools/prof_case.py --workload C5 --T 4 --cfg 3 > gpurun_out/sk8_ncu_c5_compute.csv 2>&1
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary --alt-bt 0"
STENCIL_DBG=448 timeout 300 $B --workload C4 --tile-cfg 3 > gpurun_out/sk8_bench_c4.json 2>&1
STENCIL_DBG=448 timeout 300 $B --workload C5 --tile-cfg 3 > gpurun_out/sk8_bench_c5.json 2>&1
