# cluster-pair 25v tiles (tile_cfg 1): one ncu --set full launch (C4, T = 4) for the stall attribution
python tools/prof_case.py --workload C4 --T 4 --cfg 1 > gpurun_out/pp_plain.log 2>&1 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pipe25 -s 1 -c 1 -o gpurun_out/pp_c4_cfg1 python tools/prof_case.py --workload C4 --T 4 --cfg 1 > gpurun_out/pp_ncu.log 2>&1
