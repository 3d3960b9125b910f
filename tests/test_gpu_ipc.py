"""The cross-process ST_HALO_PEER wiring with REAL CUDA IPC (two processes on this one GPU): each rank
creates its slab with halo=ST_HALO_PEER, the descriptors are all-gathered over torch.distributed (gloo),
stencil_peer_import opens the neighbour's state buffers and flag block with cudaIpcOpenMemHandle, and
stencil_peer_handshake sends rank-tagged words through both transfer paths the fused exchange uses (a
kernel's stores into the neighbour's memory, a stream-ordered cuStreamWriteValue64) and polls for the
neighbour's words from the host.  Nothing waits on the GPU for the other process (no stencil_run here:
its per-block stream waits would need a GPU per rank, see the profiling recipe)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir, mode):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    result = "fail"
    try:
        import paper_1410_3060_b200 as st
        import synth
        torch.cuda.set_device(0)
        if mode == "grid":  # Grid wires itself: export, all-gather, import, handshake, agreed verdict
            g = st.Grid(synth.K7V, 24, 20, 16, seed=3, rank=rank, nranks=world, halo=st.ST_HALO_PEER)
        else:  # the same steps by hand
            g = st.Grid(synth.K7V, 24, 20, 16, seed=3, rank=rank, nranks=world, halo=st.ST_HALO_PEER,
                        wire_peers=False)
            descs = st.exchange_peer_descriptors(g.peer_export())
            g.peer_import(*st.peer_neighbours(descs, rank))
            g.peer_handshake(timeout_ms=20000)
        info = g.info()
        dist.barrier()
        g.close()  # no block was run: nothing to wait for
        result = f"ok halo={info['halo']} own=[{info['own_z0']},{info['own_z1']})"
    except Exception as e:  # reported through the result file
        result = f"error {e}"
    finally:
        with open(os.path.join(out_dir, f"r{rank}.txt"), "w") as f:
            f.write(result)
        dist.destroy_process_group()


@pytest.mark.parametrize("world,mode", [(2, "manual"), (3, "manual"), (2, "grid"), (3, "grid")])
def test_ipc_wiring_and_handshake_two_processes(tmp_path, world, mode):
    port = _free_port()
    mp.spawn(_worker, args=(world, port, str(tmp_path), mode), nprocs=world, join=True)
    res = [open(tmp_path / f"r{r}.txt").read() for r in range(world)]
    assert all(r.startswith("ok halo=1") for r in res), res
