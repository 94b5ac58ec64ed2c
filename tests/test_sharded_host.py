"""Host-side logic of the multi-GPU path (configs[4]), on CPU.

* ns_shard_plan (the C library's tile assignment) covers every upper tile exactly once and is
  balanced to one tile.
* A world_size-2 gloo run replays the library's exchange protocol (ns_shard_chunks: own tiles cut
  into chunks -> tile-major send buffer -> one all_gather per chunk -> unpack slot s of rank q of
  chunk c = global tile (c*cs + s)*P + q, mirrored) with numpy products, and reproduces the
  unsharded Newton–Schulz step on every rank bitwise-identically (identical stop decisions need
  identical bits).
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
dist = pytest.importorskip("torch.distributed")

T = 128


@pytest.fixture(scope="module")
def nsr():
    from paper_2605_24840_b200 import build
    build.build()
    import paper_2605_24840_b200 as m
    m.load_library()
    return m


@pytest.mark.parametrize("d,P", [(1, 1), (300, 2), (1024, 3), (4096, 8), (16384, 8), (49152, 8), (49152, 5)])
def test_plan_covers_upper_triangle_once(nsr, d, P):
    n = (d + T - 1) // T
    seen = set()
    counts = []
    for r in range(P):
        t = nsr.ns_shard_plan(d, P, r)
        counts.append(len(t))
        for I, J in t:
            assert 0 <= I <= J < n
            assert (I, J) not in seen
            seen.add((int(I), int(J)))
    assert len(seen) == n * (n + 1) // 2
    assert max(counts) - min(counts) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, d, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2605_24840_b200 as nsr
        n = (d + T - 1) // T
        dp = n * T
        rng = np.random.default_rng(5)
        A = rng.standard_normal((d, d))
        A = 0.5 * (A + A.T) / np.sqrt(d)
        X = np.zeros((dp, dp))
        X[:d, :d] = A
        plans = [nsr.ns_shard_plan(d, world, r) for r in range(world)]
        n_chunks, cs = nsr.ns_shard_chunks(d, world)
        all_tiles = [None] * sum(len(p) for p in plans)
        for q_, pl in enumerate(plans):            # global tile t = local slot * P + rank
            for s_, tl in enumerate(pl):
                all_tiles[s_ * world + q_] = tuple(int(v) for v in tl)
        mine = plans[rank]

        def exchange(M):
            # the library's protocol: chunk c = local slots [c*cs, (c+1)*cs), one all_gather per chunk,
            # gathered slot s of rank q = global tile (c*cs + s)*P + q, unpacked with its mirror
            for c in range(n_chunks):
                send = np.zeros((cs, T, T))
                for s_ in range(cs):
                    if c * cs + s_ < len(mine):
                        I, J = mine[c * cs + s_]
                        send[s_] = M[I * T:(I + 1) * T, J * T:(J + 1) * T]
                out = [torch.zeros(cs * T * T, dtype=torch.float64) for _ in range(world)]
                dist.all_gather(out, torch.from_numpy(send.reshape(-1)))
                for qq in range(world):
                    if qq == rank:
                        continue
                    recv = out[qq].numpy().reshape(cs, T, T)
                    for s_ in range(cs):
                        gt = (c * cs + s_) * world + qq
                        if gt >= len(all_tiles):
                            continue
                        I, J = all_tiles[gt]
                        M[I * T:(I + 1) * T, J * T:(J + 1) * T] = recv[s_]
                        if I != J:
                            M[J * T:(J + 1) * T, I * T:(I + 1) * T] = recv[s_].T
            return M

        def own_product(P_, Q_, update):
            C = np.zeros((dp, dp))
            part = 0.0
            for I, J in mine:
                blk = P_[I * T:(I + 1) * T] @ Q_[J * T:(J + 1) * T].T
                if update:
                    blk = 1.5 * P_[I * T:(I + 1) * T, J * T:(J + 1) * T] - 0.5 * blk
                if I == J:
                    blk = np.triu(blk) + np.triu(blk, 1).T      # bitwise-symmetric diagonal tile
                C[I * T:(I + 1) * T, J * T:(J + 1) * T] = blk
                if I != J:
                    C[J * T:(J + 1) * T, I * T:(I + 1) * T] = blk.T
                if not update:
                    E = blk - (np.eye(T) * (np.arange(I * T, (I + 1) * T) < d)[:, None] if I == J else 0.0)
                    part += (1.0 if I == J else 2.0) * float(np.sum(E * E))
            return C, part

        Y, part = own_product(X, X, False)
        Y = exchange(Y)
        parts = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, torch.tensor([part], dtype=torch.float64))
        r2 = 0.0
        for pp in parts:
            r2 += float(pp[0])
        Xn, _ = own_product(X, Y, True)
        Xn = exchange(Xn)
        ref_Y = X @ X
        ref_X = 1.5 * X - 0.5 * X @ ref_Y
        ok = (np.max(np.abs(Y - ref_Y)) < 1e-13 and np.max(np.abs(Xn - ref_X)) < 1e-13
              and abs(np.sqrt(r2) - np.linalg.norm(ref_Y[:d, :d] - np.eye(d))) < 1e-11
              and np.array_equal(Y, Y.T) and np.array_equal(Xn, Xn.T))
        digest = torch.tensor([float(np.sum(Xn * np.arange(dp)[None, :])), r2], dtype=torch.float64)
        allg = [torch.zeros(2, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(allg, digest)
        same = all(torch.equal(allg[0], g) for g in allg)
        q.put((rank, bool(ok), bool(same)))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, f"error: {e!r}", False))


@pytest.mark.parametrize("d", [300, 520, 2000])
def test_gloo_two_rank_exchange(nsr, d):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, d, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, same in res:
        assert ok is True, (rank, ok)
        assert same, rank
