"""The N > 1 path's host logic on CPU: z-slab plan (stencil_plan_slab) + per-block halo exchange of the
full stored depth R*bt (also after a short remainder block), run with world_size 2 (and 3) over torch.distributed `gloo` processes.  Each rank advances its slab
with the oracle on its stored planes (halo planes act as fixed ghosts during a block, exact for the
owned planes by the R-per-step cone argument) and exchanges the R*b boundary planes of the new levels
after every block -- the schedule runtime.cu runs with NCCL.  The concatenated owned planes must equal
the global oracle run bitwise (the same point formula in the same order)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import paper_1410_3060_b200 as st
import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _exchange(arr, plan, rank, world, depth, R):
    """Swap `depth` boundary planes with z-neighbours (gloo send/recv), in place on the stored box."""
    z0 = plan["store_z0"]
    lo = plan["own_z0"] if rank > 0 else R
    hi = plan["own_z1"] if rank < world - 1 else None
    reqs = []
    bufs = []
    if rank > 0:
        send = torch.from_numpy(np.ascontiguousarray(arr[lo - z0: lo - z0 + depth]))
        recv = torch.empty_like(send)
        reqs += [dist.isend(send, rank - 1), dist.irecv(recv, rank - 1)]
        bufs.append((lo - z0 - depth, recv))
    if rank < world - 1:
        send = torch.from_numpy(np.ascontiguousarray(arr[hi - z0 - depth: hi - z0]))
        recv = torch.empty_like(send)
        reqs += [dist.isend(send, rank + 1), dist.irecv(recv, rank + 1)]
        bufs.append((hi - z0, recv))
    for r in reqs:
        r.wait()
    for off, recv in bufs:
        arr[off: off + depth] = recv.numpy()


def _worker(rank, world, port, kind, n, T, bt, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nx, ny, nz = n
        R = synth.RADIUS[kind]
        plan = st.stencil_plan_slab(nz, R, world, rank, bt)
        b_eff = plan["bt"]
        dims = synth.padded_dims(kind, nx, ny, nz)
        box = ((plan["store_z0"], plan["store_z1"]), (0, dims[1]), (0, dims[2]))
        inp = synth.make_inputs(kind, nx, ny, nz, seed=21, box=box)
        V, U = inp.V, inp.U
        nz_box = V.shape[0] - 2 * R
        for Tr in (T if isinstance(T, tuple) else (T,)):  # consecutive stencil_run calls
            left = Tr
            while left > 0:
                b = min(b_eff, left)
                oracle.run_arrays(kind, nx, ny, nz_box, V, U, inp.coef, inp.scalars, b, 1)
                _exchange(V, plan, rank, world, R * b_eff, R)
                if kind == synth.K25W:
                    _exchange(U, plan, rank, world, R * b_eff, R)
                left -= b
        z0 = plan["store_z0"]
        own = V[plan["own_z0"] - z0: plan["own_z1"] - z0]
        own_u = U[plan["own_z0"] - z0: plan["own_z1"] - z0]
        np.save(os.path.join(out_dir, f"r{rank}_v.npy"), own)
        np.save(os.path.join(out_dir, f"r{rank}_u.npy"), own_u)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind,n,T,bt,world", [
    (synth.K7V, (9, 8, 21), 7, 3, 2),
    (synth.K7C, (7, 6, 13), 9, 4, 3),
    (synth.K25V, (9, 10, 26), 5, 2, 2),
    (synth.K25W, (9, 8, 27), 5, 3, 3),
    (synth.K7V, (9, 8, 21), (3, 4, 2), 2, 3),   # remainder block, then more runs
    (synth.K7C, (7, 6, 25), (5, 7), 4, 2),
])
def test_slab_schedule_gloo_equals_global(tmp_path, kind, n, T, bt, world):
    port = _free_port()
    mp.spawn(_worker, args=(world, port, kind, n, T, bt, str(tmp_path)), nprocs=world, join=True)
    inp = synth.make_inputs(kind, *n, seed=21)
    ref_v, ref_u = oracle.run(inp, sum(T) if isinstance(T, tuple) else T, nthreads=1)
    got_v = np.concatenate([np.load(tmp_path / f"r{r}_v.npy") for r in range(world)])
    assert got_v.shape == ref_v.shape
    assert np.array_equal(got_v, ref_v)
    if kind == synth.K25W:
        got_u = np.concatenate([np.load(tmp_path / f"r{r}_u.npy") for r in range(world)])
        assert np.array_equal(got_u, ref_u)


def _desc_worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        desc = bytes([rank]) * st.ST_PEER_DESC_BYTES  # stands in for stencil_peer_export's bytes
        descs = st.exchange_peer_descriptors(desc)
        below, above = st.peer_neighbours(descs, rank)
        np.save(os.path.join(out_dir, f"d{rank}.npy"),
                np.array([-1 if below is None else below[0], -1 if above is None else above[0],
                          len(descs), min(len(d) for d in descs)]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_peer_descriptor_exchange_gloo(tmp_path, world):
    """ST_HALO_PEER's host plumbing: every rank all-gathers the descriptors and imports rank-1's as
    `below` and rank+1's as `above` (None at the ends)."""
    port = _free_port()
    mp.spawn(_desc_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        below, above, n, size = np.load(tmp_path / f"d{r}.npy")
        assert below == (r - 1 if r > 0 else -1) and above == (r + 1 if r < world - 1 else -1)
        assert n == world and size == st.ST_PEER_DESC_BYTES


def _wire_worker(rank, world, port, fail, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    calls = []
    try:
        def export():
            if fail == ("export", rank):
                raise st.StencilError(st.ST_E_CUDA, "injected export failure")
            return bytes([rank]) * st.ST_PEER_DESC_BYTES

        def import_(below, above):
            calls.append("import")
            if fail == ("import", rank):
                raise st.StencilError(st.ST_E_CUDA, "injected import failure")

        def handshake(timeout_ms):
            calls.append("handshake")
        ok, note = st.wire_peer_halos(export, import_, handshake, rank, timeout_ms=100)
        with open(os.path.join(out_dir, f"w{rank}.txt"), "w") as f:
            f.write(f"{int(ok)}|{note}|{','.join(calls)}")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("fail", [None, ("export", 1), ("import", 0), ("export", 2)])
def test_peer_wiring_failure_is_agreed_gloo(tmp_path, fail):
    """ST_HALO_PEER wiring is collective-safe: when one rank's export or import fails, every rank still
    takes part in every collective (no hang) and all ranks return the same verdict, so bench.py can
    fall back to the NCCL halo exchange on all ranks together."""
    world = 3
    port = _free_port()
    mp.spawn(_wire_worker, args=(world, port, fail, str(tmp_path)), nprocs=world, join=True)
    res = [open(tmp_path / f"w{r}.txt").read().split("|") for r in range(world)]
    oks = {r[0] for r in res}
    notes = {r[1] for r in res}
    assert len(oks) == 1 and len(notes) == 1  # one verdict, one message, on every rank
    if fail is None:
        assert oks == {"1"} and notes == {"None"}
        assert all(r[2] == "import,handshake" for r in res)
    else:
        assert oks == {"0"}
        assert f"rank {fail[1]}" in next(iter(notes))
        if fail[0] == "export":  # nobody imports when a descriptor is missing
            assert all(r[2] == "" for r in res)
