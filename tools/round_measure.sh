# One GPU call's worth of round measurements (run under gpurun from the repo root), in the order the
# profiles/ evidence is built: the GPU test suite (recording the full-size parity and oracle facts for
# the d.6 report), the bench line (C5 headline + secondaries + e2e + cpu_baseline), the reference arm,
# the bench command's ncu launch list, one ncu --set full capture of the dominant kernel, and the
# per-config d.6 report.  Each ncu pass runs only after the same command exited 0 without ncu.
# Usage: bash tools/round_measure.sh <tag>    (outputs gpurun_out/<tag>_*)
T=${1:-r02}
mkdir -p gpurun_out
STENCIL_REPORT_DIR=gpurun_out/${T}_report timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/${T}_gputests.log 2>&1
echo "rc=$?" >> gpurun_out/${T}_gputests.log
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/${T}_bench_reference.json 2> gpurun_out/${T}_bench_reference.err
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-secondary --alt-bt 0"
timeout 900 $CMD > gpurun_out/${T}_bench_short.json 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/${T}_launches.csv \
    $CMD > gpurun_out/${T}_ncu_bench.log 2>&1
timeout 600 python tools/prof_case.py --workload C5 --T 4 > gpurun_out/${T}_prof_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:pipe25 -s 1 -c 1 -o gpurun_out/${T}_c5 \
    python tools/prof_case.py --workload C5 --T 4 > gpurun_out/${T}_ncu_full.log 2>&1
timeout 900 python tools/report.py --parity gpurun_out/${T}_report/parity.json > gpurun_out/${T}_report.csv 2> gpurun_out/${T}_report.err
