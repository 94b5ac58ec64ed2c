"""The sharded path with REAL separate processes (ranks) on one GPU.

NCCL refuses two ranks on one device, so the ranks use ns_comm_init_host: the library's collectives go
through a gloo all-gather callback (torch.distributed, 127.0.0.1), while the device path is the production
one -- every rank's workspace mapped into the other processes with CUDA IPC, the product kernels' epilogues
storing their tiles and partials straight into the peers' buffers, the receivers mirroring, the
block-row init storing X_0 panels into every rank.  Each barrier is a stream synchronisation plus the host
exchange, so no kernel ever waits on another process's kernel (B200_PROFILING.md: ranks whose kernels wait
on one another must not share a GPU).  Checked: every rank's R (full entry) or row panel (rows entry) and
result record bitwise equal to the same P-rank algorithm emulated in one process, within 1e-13 of the
single-GPU ns_reflector and within 1e-10 of the oracle; a workspace that moves on one rank only between
calls (the mapping check is collective); the NCCL-free fallback protocol (NS_SHARD_P2P=0: pack, host
all-gather, unpack) on the same inputs; both mirror modes.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

import workloads  # noqa: E402
from oracle import checks, ns as ons  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem(d):
    return workloads.cfg3_dense(d=d, k=max(1, d // 16))


def _worker(rank, world, port, d, outdir, env):
    os.environ.update(env)
    import sys
    sys.path.insert(0, ROOT)
    import torch as T
    import torch.distributed as dist
    import paper_2605_24840_b200 as nsr
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    T.cuda.set_device(0)
    dev = T.device("cuda", 0)

    def allgather(b):
        out = [None] * world
        dist.all_gather_object(out, b)
        return out

    comm = nsr.ns_comm_init_host(rank, world, allgather)
    p = _problem(d)
    H = T.from_numpy(p.H).to(dev)
    nbytes = nsr.ns_workspace_bytes_sharded(d, world)
    ws = nsr.alloc_workspace(nbytes, dev)
    recs = {}
    # 1. full-H entry
    R, res = nsr.ns_reflector_sharded(comm, H, p.s, p.alpha, p.k, p.max_steps, p.tol, p.tol_mode, ws=ws, nranks=world)
    recs["full"] = (R.cpu().numpy(), res)
    # 2. rows entry, same workspace (mappings reused)
    r0, r1 = nsr.ns_shard_rows(d, world, rank)
    Rr, res = nsr.ns_reflector_sharded_rows(comm, H[r0:r1].contiguous(), d, p.s, p.alpha, p.k, p.max_steps, p.tol,
                                            p.tol_mode, ws=ws, nranks=world)
    recs["rows"] = (Rr.cpu().numpy(), res)
    # 3. the last rank's workspace moves (a new allocation); the others keep theirs: the collective mapping
    # check must re-map everywhere
    if rank == world - 1:
        keep = ws
        ws = nsr.alloc_workspace(nbytes + 4096, dev)
        del keep
    Rr2, res = nsr.ns_reflector_sharded_rows(comm, H[r0:r1].contiguous(), d, p.s, p.alpha, p.k, p.max_steps, p.tol,
                                             p.tol_mode, ws=ws, nranks=world)
    recs["rows_moved"] = (Rr2.cpu().numpy(), res)
    T.cuda.synchronize()
    np.savez(os.path.join(outdir, f"rank{rank}.npz"),
             **{f"{k}_R": v[0] for k, v in recs.items()},
             **{f"{k}_{f}": v[1][f] for k, v in recs.items() for f in ("steps", "flags", "residual", "trace", "cert")},
             r0=r0, r1=r1)
    nsr.ns_comm_destroy(comm)
    dist.barrier()
    dist.destroy_process_group()


def _run(world, d, tmp_path, env):
    import torch.multiprocessing as mp
    port = _free_port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_worker, args=(r, world, port, d, str(tmp_path), env)) for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=600)
    for pr in procs:
        if pr.is_alive():
            pr.kill()
    codes = [pr.exitcode for pr in procs]
    assert codes == [0] * world, codes
    return [dict(np.load(os.path.join(tmp_path, f"rank{r}.npz"))) for r in range(world)]


@pytest.fixture(scope="module")
def nsr():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2605_24840_b200 as m
    m.load_library()
    return m


@pytest.mark.parametrize("world,d,env", [
    (2, 2048, {}),                                   # peer stores, receivers mirror
    (3, 2304, {"NS_SHARD_MIRROR": "sender"}),        # peer stores incl. mirrors
    (2, 2048, {"NS_SHARD_P2P": "0"}),                # fallback: pack / all-gather / unpack
    (4, 1000, {}),                                   # ragged d (d_pad = 1024), 4 ranks
])
def test_processes_share_one_gpu(nsr, tmp_path, world, d, env):
    """Reference: the same P-rank algorithm emulated in one process (same 128x128-tile kernels, so the real
    processes must reproduce it bitwise) and the single-GPU path / the oracle (within rounding / 1e-10)."""
    p = _problem(d)
    Hg = torch.from_numpy(p.H).to("cuda:0")
    Re, re_ = nsr.ns_reflector_sharded_emulated(world, Hg, p.s, p.alpha, p.k, p.max_steps, p.tol, p.tol_mode)
    Re = Re.cpu().numpy()
    R1, r1 = nsr.ns_reflector(Hg, p.s, p.alpha, p.k, p.max_steps, p.tol, p.tol_mode)
    R1 = R1.cpu().numpy()
    o = ons.ns_reflector(p.H, p.s, p.alpha, p.k, p.max_steps, p.tol, p.tol_mode)
    outs = _run(world, d, tmp_path, env)
    for rank, z in enumerate(outs):
        r0_, r1_ = int(z["r0"]), int(z["r1"])
        assert (r0_, r1_) == (d // world * rank, d // world * (rank + 1))
        for case in ("full", "rows", "rows_moved"):
            Rk = z[f"{case}_R"]
            sl = slice(None) if case == "full" else slice(r0_, r1_)
            assert np.array_equal(Rk, Re[sl]), (rank, case)
            assert np.max(np.abs(Rk - R1[sl])) <= 1e-13, (rank, case)
            for f in ("steps", "flags", "cert", "residual", "trace"):
                assert z[f"{case}_{f}"] == re_[f], (rank, case, f)
            assert int(z[f"{case}_steps"]) == r1["steps"] == o["steps"]
            assert int(z[f"{case}_cert"]) == p.k
    assert checks.frob_per_sqrt_d(outs[0]["full_R"], o["R"]) <= 1e-10
