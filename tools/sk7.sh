# skewed tiles without the dependency (STENCIL_DBG=192: no flag wait, no fence; wrong results) next to the
# default tile: one ncu --set full launch each (C4, T = 4), to compare their per-step costs
python tools/prof_case.py --workload C4 --T 4 --cfg 3 > gpurun_out/sk7_plain.log 2>&1 || exit 1
STENCIL_DBG=192 timeout 600 ncu --set full --clock-control none --import-source on -k regex:pipe25 -s 1 -c 1 -o gpurun_out/sk7_c4_cfg3_nowait python tools/prof_case.py --workload C4 --T 4 --cfg 3 > gpurun_out/sk7_ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pipe25 -s 1 -c 1 -o gpurun_out/sk7_c4_cfg0 python tools/prof_case.py --workload C4 --T 4 --cfg 0 > gpurun_out/sk7_ncu2.log 2>&1
