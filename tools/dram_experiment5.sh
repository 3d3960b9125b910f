M="--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -s 1 -c 1 --csv"
python tools/prof_case.py --workload C4 --T 4 > gpurun_out/dv_plain.log 2>&1 || exit 1
ncu $M -k regex:pipe25 python tools/prof_case.py --workload C4 --T 4 > gpurun_out/dv_c4.csv 2>&1
ncu $M -k regex:pipe25 python tools/prof_case.py --workload C5 --T 4 > gpurun_out/dv_c5.csv 2>&1
ncu $M -k regex:pipe_kernel python tools/prof_case.py --workload C2 --bt 4 --T 8 > gpurun_out/dv_c2.csv 2>&1
for w in C4 C5 C2; do timeout 300 python bench.py --workload $w --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --no-secondary --alt-bt 0 > gpurun_out/dv_bench_$w.json 2>&1; done
