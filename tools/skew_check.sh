# Skewed 25v tiles (tile_cfg 3): bitwise/oracle tests, then sustained rate (release every
# STENCIL_XG steps) and one ncu launch next to the default plan.  Usage: bash tools/skew_check.sh <tag>
T=${1:-sk}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_25v_bt2.py -x -q > gpurun_out/${T}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${T}_tests.log
tail -1 gpurun_out/${T}_tests.log | grep -q "rc=0" || exit 1
for xg in 1 4 8; do
  STENCIL_XG=$xg timeout 600 python bench.py --workload C4 --tile-cfg 3 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary --alt-bt 0 > gpurun_out/${T}_bench_C4_cfg3_xg$xg.json 2>&1
done
M="--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum,l1tex__m_xbar2l1tex_read_bytes.sum --clock-control none -s 1 -c 1 --csv"
for xg in 1 4 8; do
  STENCIL_XG=$xg timeout 600 ncu $M -k regex:pipe25 python tools/prof_case.py --workload C4 --T 4 --cfg 3 > gpurun_out/${T}_ncu_C4_cfg3_xg$xg.csv 2>&1
done
STENCIL_XG=4 timeout 600 ncu --set full --clock-control none --import-source on -k regex:pipe25 -s 1 -c 1 -o gpurun_out/${T}_c4_cfg3 python tools/prof_case.py --workload C4 --T 4 --cfg 3 > gpurun_out/${T}_ncu_full.log 2>&1
