"""Distinct handles may be used concurrently (include/stencil.h conventions): grids created
from host arrays in worker threads on their own streams while other grids run -- the pattern of
bench.py's pipelined end-to-end measurement -- give bitwise the results of the sequential runs.  (One handle is never used by two
threads at once here: a handle is not reentrant; the library refuses that with ST_E_STATE.)"""
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
import torch

import paper_1410_3060_b200 as st
import synth

pytestmark = pytest.mark.gpu

CASES = [(synth.K7V, (48, 40, 36), 9), (synth.K25W, (70, 20, 30), 5), (synth.K25V, (66, 17, 29), 4)]


def _host_grid(kind, n, seed, stream=None, variant=st.ST_VARIANT_PIPE):
    inp = synth.make_inputs(kind, *n, seed=seed)
    coeff = list(inp.scalars) + list(inp.coef)
    u0 = inp.U if kind in synth.WAVE_KINDS else None
    return st.Grid(kind, *n, v0=inp.V, u0=u0, coeff=coeff, stream=stream, variant=variant)


@pytest.mark.parametrize("kind,n,T", CASES)
def test_pipelined_create_matches_sequential(kind, n, T):
    seeds = [3, 4, 5, 6]
    ref = []
    for sd in seeds:
        with _host_grid(kind, n, sd) as g:
            g.run(T)
            ref.append(g.read(0))
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    dev = torch.cuda.current_device()

    def create(k):
        torch.cuda.set_device(dev)
        return _host_grid(kind, n, seeds[k], stream=streams[k % 2])

    got = []
    with ThreadPoolExecutor(1) as ex:
        fut = ex.submit(create, 0)
        for k in range(len(seeds)):
            g = fut.result()
            if k + 1 < len(seeds):
                fut = ex.submit(create, k + 1)
            g.run(T)
            got.append(g.read(0))
            g.close()
    for a, b in zip(got, ref):
        assert np.array_equal(a, b)


def test_threads_on_distinct_handles():
    kind, n, T = synth.K7V, (40, 33, 37), 6
    ref = {}
    for sd in (1, 2, 3):
        with _host_grid(kind, n, sd) as g:
            g.run(T)
            ref[sd] = g.read(0)
    out, errs = {}, []
    dev = torch.cuda.current_device()

    def work(sd):
        try:
            torch.cuda.set_device(dev)
            with _host_grid(kind, n, sd, stream=torch.cuda.Stream()) as g:
                for _ in range(T):
                    g.run(1)
                out[sd] = g.read(0)
        except Exception as e:  # surfaced below
            errs.append(e)
    th = [threading.Thread(target=work, args=(sd,)) for sd in (1, 2, 3)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for sd in (1, 2, 3):
        assert np.array_equal(out[sd], ref[sd])
