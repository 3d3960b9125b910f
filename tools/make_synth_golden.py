"""Write tests/golden/synth_golden.txt: frozen values of the synth.h generator.

Computed with the pure-numpy restatement synth.numpy_unit (not the C fill), so the golden file
freezes the documented definition in synth.h's header.  Run: python tools/make_synth_golden.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402

CASES = [(0, 0), (1, 0), (14103060, 0), (14103060, 1), (14103060, 2), (14103060, 8), (7, 14)]
IDX = [0, 1, 2, 3, 1000, 2 ** 31 + 5, 2 ** 40 + 17]


def main():
    out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                       "tests", "golden", "synth_golden.txt")
    with open(out, "w") as f:
        f.write("# synth.h golden values: seed stream idx u(hex)   -- written by tools/make_synth_golden.py\n")
        for seed, stream in CASES:
            u = synth.numpy_unit(seed, stream, np.array(IDX, dtype=np.uint64))
            for i, v in zip(IDX, u):
                f.write(f"{seed} {stream} {i} {float(v).hex()}\n")
    print("wrote", out)


if __name__ == "__main__":
    main()
