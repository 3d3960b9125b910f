# One GPU call's worth of round measurements (run under gpurun from the repo root):
# default-plan sweep over every workload, the bench line, and the bench command's ncu launch list.
set -e
mkdir -p gpurun_out
python tools/sweep.py --workloads C1,C2,C3,C4,C3A,C5 --variants 3 --bts 0 --reps 3 > gpurun_out/sweep_default.jsonl 2>&1
python tools/sweep.py --workloads C2 --variants 3 --bts 1,2,3 --reps 3 >> gpurun_out/sweep_default.jsonl 2>&1
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_short.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_bench.log 2>&1
