# One GPU call's worth of round measurements (run under gpurun from the repo root), in the order the
# profiles/ evidence is built: the bench line, the reference arm, the bench command's ncu launch list,
# one ncu --set full capture of the dominant kernel, the per-config report (with board power), the
# power probe and the end-to-end timeline.  Each ncu pass runs only after its command exited 0 without ncu.
set -e
mkdir -p gpurun_out
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_short.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_bench.log 2>&1
python tools/prof_case.py --workload C2 --bt 3 --T 9 > /dev/null
ncu --set full --clock-control none --import-source on -k regex:pipe_kernel -s 2 -c 1 -o gpurun_out/c2_bt3 \
    python tools/prof_case.py --workload C2 --bt 3 --T 9 > gpurun_out/ncu_full.log 2>&1
python tools/report.py > gpurun_out/report.csv 2> gpurun_out/report.err
python tools/power_probe.py > gpurun_out/power_probe.json 2>&1
python tools/e2e_probe.py > gpurun_out/e2e_probe.log 2>&1
