M="--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:pipe25 -s 1 -c 1 --csv"
python tools/prof_case.py --workload C5 --T 4 > gpurun_out/dx_plain.log 2>&1 || exit 1
for tb in 43 11 4 1; do STENCIL_TILE_BLOCK=$tb ncu $M python tools/prof_case.py --workload C5 --T 4 > gpurun_out/dx_tb$tb.csv 2>&1; done
STENCIL_SCHED=0 ncu $M python tools/prof_case.py --workload C5 --T 4 > gpurun_out/dx_dyn.csv 2>&1
ncu $M python tools/prof_case.py --workload C5 --T 4 --zchunk 128 > gpurun_out/dx_zc128.csv 2>&1
ncu $M python tools/prof_case.py --workload C4 --T 4 > gpurun_out/dx_c4.csv 2>&1
ncu $M python tools/prof_case.py --workload C5 --T 4 --bt 1 > gpurun_out/dx_c5bt1.csv 2>&1
