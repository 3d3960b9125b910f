"""The multi-GPU z-slab plan on one GPU: a handle holding all P slabs
("loopback": halos exchanged by device copies after every fused block, the same plan and kernels as the
NCCL path; or, with ST_HALO_PEER, stored by the kernel straight into the neighbour slab -- the fused
exchange of SURVEY NEXT-2) must reproduce the single-slab run bitwise (G4 across slab counts) and match
the oracle."""
import numpy as np
import pytest

import oracle
import paper_1410_3060_b200 as st
import synth
from gpu_common import WAVES, assert_parity

pytestmark = pytest.mark.gpu


def run(kind, n, T, **kw):
    with st.Grid(kind, *n, seed=31, **kw) as g:
        for t in (T if isinstance(T, tuple) else (T,)):  # a tuple = consecutive stencil_run calls
            g.run(t)
        new = g.read(0)
        old = g.read(1) if kind in WAVES else None
        info = g.info()
    return new, old, info


def run_ranks(gs, T):
    """Run ST_HALO_PEER ranks emulated as handles of this process: every rank's host waits for its
    neighbours' block flags before enqueuing its next block (runtime.cu peer_wait), so each rank runs
    T (an int, or a tuple of consecutive runs) from its own host thread, as separate processes do."""
    import threading

    import torch
    errs = []

    def drive(g):
        try:
            torch.cuda.set_device(0)
            for t in (T if isinstance(T, tuple) else (T,)):
                g.run(t)
            g.sync()
        except Exception as e:  # noqa: BLE001 -- reported below
            errs.append(e)
    th = [threading.Thread(target=drive, args=(g,)) for g in gs]
    for x in th:
        x.start()
    for x in th:
        x.join(timeout=120)
    assert not errs and not any(x.is_alive() for x in th), errs


CASES = [
    (synth.K7C, (40, 33, 37), 11),
    (synth.K7V, (40, 33, 37), 9),
    (synth.K25W, (70, 20, 41), 6),
    (synth.K25V, (70, 20, 41), 6),
    (synth.K25WA, (70, 20, 41), 6),
]


@pytest.mark.parametrize("kind,n,T", CASES)
@pytest.mark.parametrize("P", [2, 3, 5])
def test_loopback_slabs_bitwise_equal_single(kind, n, T, P):
    ref = run(kind, n, T)
    for variant, bt in ((st.ST_VARIANT_PIPE, 0), (st.ST_VARIANT_PIPE, 2 if synth.RADIUS[kind] == 1 else 1),
                        (st.ST_VARIANT_STREAM, 1), (st.ST_VARIANT_NAIVE, 0)):
        got = run(kind, n, T, nranks=P, local_slabs=P, variant=variant, bt=bt)
        assert got[2]["nranks"] == P and got[2]["local_slabs"] == P
        assert np.array_equal(got[0], ref[0]), (variant, bt)
        if kind in WAVES:
            assert np.array_equal(got[1], ref[1]), (variant, bt)


@pytest.mark.parametrize("kind,n,T", CASES)
@pytest.mark.parametrize("halo", [st.ST_HALO_COPY, st.ST_HALO_PEER])
def test_loopback_slabs_oracle_parity(kind, n, T, halo):
    inp = synth.make_inputs(kind, *n, seed=31)
    o_new, o_old = oracle.run(inp, T)
    g_new, g_old, info = run(kind, n, T, nranks=4, local_slabs=4, halo=halo)
    assert info["halo"] == halo
    assert_parity(kind, g_new, g_old, o_new, o_old, inp.R, 1e-12, inputs=inp)


def test_bt_clamped_to_thinnest_slab():
    # 25-point, nz = 16 over 4 slabs of 4 planes: R*bt <= 4 forces bt = 1
    new, _, info = run(synth.K25V, (20, 20, 16), 3, nranks=4, local_slabs=4, bt=1)
    assert info["bt"] == 1
    # 7-point, nz = 9 over 3 slabs of 3 planes: bt clamped to 3
    _, _, info = run(synth.K7C, (20, 20, 9), 5, nranks=3, local_slabs=3, bt=8)
    assert info["bt"] == 3


def test_weak_shape_medium():
    """7v 128 x 128 x (64 * 4) over 4 slabs, T = 20, default plan: bitwise equal to one slab."""
    n = (128, 128, 256)
    a = run(synth.K7V, n, 20)
    b = run(synth.K7V, n, 20, nranks=4, local_slabs=4)
    assert np.array_equal(a[0], b[0])


@pytest.mark.parametrize("kind,n,T", CASES)
def test_overlap_schedule_equals_bulk_synchronous(kind, n, T, monkeypatch):
    """Halo-first schedule (edge kernels, exchange on a comm stream, interior kernel; STENCIL_OVERLAP=1) ==
    one launch per slab followed by the exchange (the default), bitwise."""
    monkeypatch.setenv("STENCIL_OVERLAP", "1")
    a = run(kind, n, T, nranks=3, local_slabs=3)
    monkeypatch.delenv("STENCIL_OVERLAP")
    b = run(kind, n, T, nranks=3, local_slabs=3)
    assert np.array_equal(a[0], b[0])
    assert a[2]["launches"] > b[2]["launches"]  # the split schedule launches edge + interior kernels


def test_invalid_slab_options():
    with pytest.raises(st.StencilError):
        st.Grid(synth.K7V, 8, 8, 8, seed=1, nranks=2, local_slabs=3)
    with pytest.raises(st.StencilError):
        st.Grid(synth.K25V, 8, 8, 12, seed=1, nranks=4, local_slabs=4)  # 3-plane slabs < R = 4


@pytest.mark.parametrize("kind,n,T", CASES)
@pytest.mark.parametrize("P", [2, 3, 5])
def test_peer_halo_bitwise_equal_single(kind, n, T, P):
    """Fused halo exchange (ST_HALO_PEER): one launch per slab and block, the kernel stores the
    neighbours' halo planes itself; bitwise equal to one slab for every bt the slabs allow."""
    ref = run(kind, n, T)
    R = synth.RADIUS[kind]
    for bt in sorted({0, 1, 2 if R == 1 else 1, 3 if R == 1 else 1}):
        got = run(kind, n, T, nranks=P, local_slabs=P, halo=st.ST_HALO_PEER, bt=bt)
        info = got[2]
        assert info["halo"] == st.ST_HALO_PEER
        b = info["bt"]
        assert info["launches"] == P * -(-T // b)  # no edge/interior split, no copies
        assert np.array_equal(got[0], ref[0]), bt
        if kind in WAVES:
            assert np.array_equal(got[1], ref[1]), bt


@pytest.mark.parametrize("kind,bt", [(synth.K7C, 4), (synth.K7V, 2), (synth.K7V, 3)])
@pytest.mark.parametrize("halo", [0, 1])
def test_remainder_block_then_next_run(kind, bt, halo):
    """run(T1) ending in a short block (T1 mod bt != 0) followed by run(T2): the halos after the short
    block must still cover the full R*bt depth the next run's first block reads."""
    n = (40, 33, 37)
    T = (bt + 1, 2 * bt, bt - 1 if bt > 1 else 1)
    ref = run(kind, n, T)
    got = run(kind, n, T, nranks=3, local_slabs=3, bt=bt, halo=halo)
    assert got[2]["bt"] == bt
    assert np.array_equal(got[0], ref[0])


def test_peer_halo_needs_pipe_variant():
    with pytest.raises(st.StencilError):
        st.Grid(synth.K7V, 16, 16, 16, seed=1, nranks=2, local_slabs=2, halo=st.ST_HALO_PEER,
                variant=st.ST_VARIANT_STREAM)


@pytest.mark.parametrize("kind,n,T", [CASES[1], CASES[3], (synth.K7V, (40, 33, 37), (5, 4)),
                                      (synth.K25W, (70, 20, 41), (3, 2))])
@pytest.mark.parametrize("P", [2, 3])
def test_peer_ranks_as_handles_in_one_process(kind, n, T, P):
    """The one-slab-per-rank ST_HALO_PEER protocol (descriptor export/import, remote stores into the
    neighbour's buffers, stream-ordered flag write / wait per block) with P ranks emulated as P handles
    of this process on their own streams and host threads (descriptors from the same process are used
    without IPC).  Each rank's host waits for its neighbours' block flags before enqueuing a block -- no
    kernel or stream waits on another rank.  Owned planes of all ranks == one slab, bitwise."""
    import torch
    ref = run(kind, n, T)
    streams = [torch.cuda.Stream() for _ in range(P)]
    gs = [st.Grid(kind, *n, seed=31, rank=r, nranks=P, halo=st.ST_HALO_PEER, wire_peers=False,
                  stream=streams[r]) for r in range(P)]
    try:
        descs = [g.peer_export() for g in gs]
        assert all(len(d) == st.ST_PEER_DESC_BYTES for d in descs)
        for r, g in enumerate(gs):
            g.peer_import(*st.peer_neighbours(descs, r))
        # handshake: rank 0 alone times out (its neighbour has not stored yet); once every rank has
        # posted its words, every rank finds both neighbours' words
        with pytest.raises(st.StencilError):
            gs[0].peer_handshake(timeout_ms=20)
        for g in gs[1:]:
            try:
                g.peer_handshake(timeout_ms=0)
            except st.StencilError:
                pass
        for g in gs:
            g.peer_handshake(timeout_ms=2000)
        run_ranks(gs, T)
        new = np.zeros(gs[0].padded_shape)
        old = np.zeros(gs[0].padded_shape)
        for g in gs:
            g.read(0, out=new)
            if kind in WAVES:
                g.read(1, out=old)
        assert np.array_equal(new, ref[0])
        if kind in WAVES:
            assert np.array_equal(old, ref[1])
        assert gs[0].info()["halo"] == st.ST_HALO_PEER
    finally:
        for g in gs:
            g.close()


def test_peer_import_validates():
    a = st.Grid(synth.K7V, 16, 16, 16, seed=1, rank=0, nranks=2, halo=st.ST_HALO_PEER, wire_peers=False)
    b = st.Grid(synth.K7V, 16, 16, 16, seed=1, rank=1, nranks=2, halo=st.ST_HALO_PEER, wire_peers=False)
    try:
        da, db = a.peer_export(), b.peer_export()
        with pytest.raises(st.StencilError):
            a.peer_import(None, None)       # rank 0 of 2 needs an `above`
        with pytest.raises(st.StencilError):
            a.peer_import(None, da)         # its own descriptor is not rank 1's
        with pytest.raises(st.StencilError):
            a.run(1)                        # not wired yet
        a.peer_import(None, db)
        b.peer_import(da, None)
        with pytest.raises(st.StencilError):
            b.peer_import(da, None)         # twice
    finally:
        a.close()
        b.close()


@pytest.mark.parametrize("halo", [0, 1])
@pytest.mark.parametrize("P", [2, 3])
def test_wave_bt2_slabs(halo, P):
    """The leapfrog at bt = 2 (four state buffers, BOTH time levels exchanged / forwarded after every
    block) over z-slabs == one slab, bitwise, including a remainder block and a second run."""
    n, T = (70, 20, 41), (5, 2)
    ref = run(synth.K25W, n, T, bt=2, variant=st.ST_VARIANT_PIPE)
    got = run(synth.K25W, n, T, nranks=P, local_slabs=P, bt=2, halo=halo)
    assert got[2]["bt"] == 2 and ref[2]["bt"] == 2
    assert np.array_equal(got[0], ref[0]) and np.array_equal(got[1], ref[1])


@pytest.mark.parametrize("kind,n,T,bt", [(synth.K7V, (40, 33, 37), 7, 3), (synth.K25W, (70, 20, 41), 5, 1),
                                         (synth.K25V, (70, 20, 41), 4, 1)])
@pytest.mark.parametrize("P", [2, 3])
def test_host_slab_inputs(kind, n, T, bt, P):
    """st_opts.host_slab: each rank passes host arrays holding only its stored planes
    [store_z0, store_z1) (stencil_plan_slab) -- a rank never holds the global inputs -- and reads back
    its owned planes with stencil_read_planes.  Ranks emulated as handles of this process (ST_HALO_PEER
    protocol as above); owned planes of all ranks == a single slab created from the global arrays,
    bitwise; stencil_write with a local array round-trips."""
    import torch
    R = synth.RADIUS[kind]
    inp = synth.make_inputs(kind, *n, seed=7)
    coeff = list(inp.scalars) + list(inp.coef)
    u0 = inp.U if kind in WAVES else None
    with st.Grid(kind, *n, v0=inp.V, u0=u0, coeff=coeff, bt=bt) as g:
        g.run(T)
        ref = g.read(0)
    dims = synth.padded_dims(kind, *n)
    streams = [torch.cuda.Stream() for _ in range(P)]
    gs, locs = [], []
    try:
        for r in range(P):
            pl = st.stencil_plan_slab(n[2], R, P, r, bt)
            box = ((pl["store_z0"], pl["store_z1"]), (0, dims[1]), (0, dims[2]))
            loc = synth.make_inputs(kind, *n, seed=7, box=box)
            locs.append((pl["store_z0"], loc.V))
            gs.append(st.Grid(kind, *n, v0=loc.V, u0=loc.U if kind in WAVES else None,
                              coeff=list(loc.scalars) + list(loc.coef), bt=bt, rank=r, nranks=P,
                              halo=st.ST_HALO_PEER, wire_peers=False, stream=streams[r], host_slab=True))
        descs = [g.peer_export() for g in gs]
        for r, g in enumerate(gs):
            g.peer_import(*st.peer_neighbours(descs, r))
        for g in gs:  # post every rank's words first, then poll
            try:
                g.peer_handshake(timeout_ms=0)
            except st.StencilError:
                pass
        for g in gs:
            g.peer_handshake(timeout_ms=2000)
        run_ranks(gs, T)
        for r, g in enumerate(gs):
            i = g.info()
            z0, z1 = i["own_z0"], i["own_z1"]
            assert np.array_equal(g.read_planes(0, z0, z1), ref[z0:z1])
        for g, (s0, lv) in zip(gs, locs):  # stencil_write from a local array round-trips
            g.sync()
            g.write(0, lv)
            i = g.info()
            assert np.array_equal(g.read_planes(0, i["own_z0"], i["own_z1"]), lv[i["own_z0"] - s0:i["own_z1"] - s0])
        # a local array of the wrong size is rejected by the binding
        pl = st.stencil_plan_slab(n[2], R, P, 0, bt)
        with pytest.raises(ValueError):
            st.Grid(kind, *n, v0=inp.V, u0=u0, coeff=coeff, bt=bt, rank=0, nranks=P, halo=st.ST_HALO_PEER,
                    wire_peers=False, host_slab=True)
    finally:
        for g in gs:
            g.close()


def test_host_slab_needs_explicit_bt_and_ranks():
    inp = synth.make_inputs(synth.K7V, 8, 8, 8, seed=1)
    with pytest.raises(ValueError):  # a single rank: nothing to slice
        st.Grid(synth.K7V, 8, 8, 8, v0=inp.V, coeff=list(inp.coef), bt=2, host_slab=True)
    pl = st.stencil_plan_slab(8, 1, 2, 0, 2)
    loc = synth.make_inputs(synth.K7V, 8, 8, 8, seed=1, box=((pl["store_z0"], pl["store_z1"]), (0, 10), (0, 10)))
    with pytest.raises(ValueError):  # bt = 0: the stored range is not known in advance
        st.Grid(synth.K7V, 8, 8, 8, v0=loc.V, coeff=list(loc.coef), rank=0, nranks=2, halo=st.ST_HALO_PEER,
                wire_peers=False, host_slab=True)
    # the library enforces the same rule for C callers (raw ABI call, no binding-side check)
    import ctypes
    from paper_1410_3060_b200 import _binding as B
    o = st.stencil_opts_default()
    o.nranks, o.rank, o.halo, o.host_slab = 2, 0, st.ST_HALO_PEER, 1  # bt = 0
    arrs = [np.ascontiguousarray(c) for c in inp.coef]
    ptrs = (ctypes.c_void_p * 7)(*[a.ctypes.data for a in arrs])
    h = ctypes.c_void_p()
    rc = B.lib().stencil_create(ctypes.byref(h), synth.K7V, 8, 8, 8, ctypes.cast(ptrs, ctypes.c_void_p), 7,
                                np.ascontiguousarray(inp.V).ctypes.data, None, ctypes.byref(o))
    assert rc == st.ST_E_INVAL and "host_slab" in st.stencil_last_error()

