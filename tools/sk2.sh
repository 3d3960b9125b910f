python tools/dbg_skew.py 130 37 41 2 > gpurun_out/sk2_a.log 2>&1
STENCIL_DBG=32 python tools/dbg_skew.py 130 37 41 2 > gpurun_out/sk2_b.log 2>&1
python tools/dbg_skew.py 24 60 20 2 > gpurun_out/sk2_c.log 2>&1
python tools/dbg_skew.py 24 10 20 2 > gpurun_out/sk2_d.log 2>&1
python tools/dbg_skew.py 130 37 41 2 1000 > gpurun_out/sk2_e.log 2>&1
