import sys, os, json, statistics
sys.path.insert(0, os.getcwd())
import torch
import paper_1410_3060_b200 as st
import synth
torch.cuda.set_device(0)
s = torch.cuda.current_stream()
for kind, n, T in [(1, 8, 1), (1, 8, 10), (1, 8, 50), (1, 64, 10), (1, 96, 10), (1, 128, 10), (1, 192, 10), (2, 64, 10), (2, 128, 10), (3, 64, 10), (3, 96, 10), (4, 64, 10), (4, 96, 10), (2, 64, 100)]:
    for variant, bt, cfg in [(4, 1, 0), (4, 1, 2), (3, 0, 0)]:  # coop: one sweep per barrier / blocked; pipe
        if cfg == 2 and kind not in (1, 2):
            continue
        g = st.Grid(kind, n, n, n, seed=1, variant=variant, bt=bt, tile_cfg=cfg)
        g.run(T); g.sync()
        ts = []
        for _ in range(20):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s); g.run(T); e1.record(s); e1.synchronize(); ts.append(e0.elapsed_time(e1))
        ms = statistics.median(ts)
        print(json.dumps({"kind": kind, "n": n, "T": T, "variant": variant, "cfg": cfg, "tile": [g.info()["tile_x"], g.info()["zchunk"]], "bt": g.info()["bt"], "us": round(ms * 1e3, 1),
                          "glups": round(n**3 * T / ms / 1e6, 1)}), flush=True)
        g.close()
