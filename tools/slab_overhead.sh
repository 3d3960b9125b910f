for w in C2 C4; do for P in 2 4 8; do for h in copy peer; do
python bench.py --workload $w --slabs $P --halo $h --steps 3 --warmup 3 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', $P, '$h', round(d['value'],1), d['gpu_launches'], d['config']['parallelism'])"
done; done; done
python bench.py --workload C2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C2 1', round(d['value'],1))"
python bench.py --workload C4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C4 1', round(d['value'],1))"
