# 7-point variable kind at b_t = 5 (TMEM window, 2x1 cells): GPU parity tests, sustained C2 next to b_t = 4, one ncu launch
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/bt5_tests.log 2>&1; echo rc=$? >> gpurun_out/bt5_tests.log
B="python bench.py --workload C2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary --alt-bt 0"
for c in "--bt 5" "--bt 5 --tile-cfg 1" "--bt 4"; do timeout 300 $B $c > "gpurun_out/bt5_bench_${c// /_}.json" 2>&1; done
M="--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -s 1 -c 1 --csv"
timeout 300 ncu $M -k regex:pipe_kernel python tools/prof_case.py --workload C2 --bt 5 --T 10 > gpurun_out/bt5_ncu.csv 2>&1
