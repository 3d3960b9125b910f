"""Cooperative kernel at small grids: one sweep per grid barrier (tile_cfg 0) vs temporal blocking in
shared memory with rounds of 5 levels (tile_cfg 2).  python tools/coop_tb_sweep.py"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import statistics, torch, paper_1410_3060_b200 as st
torch.cuda.set_device(0); s = torch.cuda.current_stream()
for kind, n, T in [(1, 64, 10), (1, 64, 100), (2, 64, 10), (1, 32, 10), (1, 96, 10)]:
    for cfg in (0, 2):
        g = st.Grid(kind, n, n, n, seed=1, variant=4, tile_cfg=cfg)
        g.run(T); g.sync(); ts = []
        for _ in range(30):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s); g.run(T); e1.record(s); e1.synchronize(); ts.append(e0.elapsed_time(e1))
        ms = statistics.median(ts)
        print(f"kind={kind} n={n} T={T} cfg={cfg} us={ms*1e3:.1f} glups={n**3*T/ms/1e6:.1f}", flush=True)
        g.close()
