M="--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:pipe_kernel -s 1 -c 1 --csv"
python tools/prof_case.py --workload C2 --bt 4 --T 8 > gpurun_out/dz_plain.log 2>&1 || exit 1
ncu $M python tools/prof_case.py --workload C2 --bt 4 --T 8 > gpurun_out/dz_c2.csv 2>&1
STENCIL_SCHED=0 ncu $M python tools/prof_case.py --workload C2 --bt 4 --T 8 > gpurun_out/dz_c2_dyn.csv 2>&1
for tb in 4 19; do STENCIL_TILE_BLOCK=$tb ncu $M python tools/prof_case.py --workload C2 --bt 4 --T 8 > gpurun_out/dz_c2_tb$tb.csv 2>&1; done
ncu $M python tools/prof_case.py --workload C2 --bt 4 --T 8 --zchunk 512 > gpurun_out/dz_c2_zc512.csv 2>&1
ncu $M python tools/prof_case.py --workload C3 --bt 1 --T 3 > gpurun_out/dz_c3.csv 2>&1
