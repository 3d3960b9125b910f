nvidia-smi --query-gpu=power.limit,enforced.power.limit,power.max_limit,power.default_limit --format=csv > gpurun_out/pw_limits.csv
nvidia-smi --query-gpu=timestamp,power.draw,power.draw.average,power.draw.instant,clocks.sm,clocks.mem,temperature.gpu,clocks_event_reasons.active --format=csv -lms 100 > gpurun_out/pw_trace.csv &
P=$!
sleep 1
timeout 200 python tools/sweep.py --workloads C2 --variants 3 --bts 3 --T 600 --reps 2 > gpurun_out/pw_sweep.json
timeout 200 python tools/sweep.py --workloads C3 --variants 3 --bts 1 --T 600 --reps 2 >> gpurun_out/pw_sweep.json
kill $P
