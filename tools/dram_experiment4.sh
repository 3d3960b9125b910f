M="--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:pipe25 -s 1 -c 1 --csv"
python tools/prof_case.py --workload C4 --T 4 > gpurun_out/dw_plain.log 2>&1 || exit 1
for sk in 0 2000 5000 20000; do STENCIL_SKEW_NS=$sk ncu $M python tools/prof_case.py --workload C4 --T 4 > gpurun_out/dw_sk$sk.csv 2>&1; done
