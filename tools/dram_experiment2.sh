M="--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:pipe25 -s 1 -c 1 --csv"
python tools/prof_case.py --workload C5 --T 4 > gpurun_out/dy_plain.log 2>&1 || exit 1
for pr in 1 2 3; do STENCIL_TMA_PROMO=$pr ncu $M python tools/prof_case.py --workload C5 --T 4 > gpurun_out/dy_pr$pr.csv 2>&1; done
for pr in 2 3; do STENCIL_TMA_PROMO=$pr timeout 300 python bench.py --workload C5 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-secondary --alt-bt 0 > gpurun_out/dy_bench_pr$pr.json 2>&1; done
