"""Multi-rank host logic on CPU (gloo, world_size 2 and 3): the z-slab plan of the
library (dg_slab_plan), its halo packer (dg_halo_pack_host, same index map as the
device pack kernel) and the documented two-phase message order ("up" then "down",
include/dg.h), exchanged over torch.distributed gloo.  Every rank checks that the
received planes are exactly the neighbouring ranks' face layers of the global
vector (2 layers per face for the Hermite-like basis)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _layers(U, cz, layers):
    """[cxy][l][j][i] planes of global cells at z index cz (U: [cz][cy][cx][k][j][i])."""
    plane = U[cz]                       # [cy][cx][k][j][i]
    Ny, Nx = plane.shape[:2]
    return plane[:, :, layers].reshape(Ny * Nx, len(layers), -1).reshape(-1)


def _worker(rank, world, port, cases, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1907_08492_b200 as P
    try:
        for (p, basis, N, bc) in cases:
            n = p + 1
            Nx, Ny, Nz = N
            rng = np.random.default_rng(1234)
            U = rng.uniform(-1, 1, (Nz, Ny, Nx, n, n, n))
            plan = P.slab_plan(Nz, world, rank, bc, p, basis)
            zb, ze, lo, hi, NL = plan["z_begin"], plan["z_end"], plan["lo_peer"], plan["hi_peer"], plan["NL"]
            slab = U[zb:ze].reshape(-1)
            send_lo, send_hi = P.halo_pack_host(slab, p, basis, Nx, Ny, ze - zb)
            recv_lo = torch.zeros(send_lo.size, dtype=torch.float64)
            recv_hi = torch.zeros(send_hi.size, dtype=torch.float64)
            reqs = []
            # phase "up"
            if hi >= 0:
                reqs.append(dist.isend(torch.from_numpy(send_hi), hi))
            if lo >= 0:
                reqs.append(dist.irecv(recv_lo, lo))
            for r in reqs:
                r.wait()
            reqs = []
            # phase "down"
            if lo >= 0:
                reqs.append(dist.isend(torch.from_numpy(send_lo), lo))
            if hi >= 0:
                reqs.append(dist.irecv(recv_hi, hi))
            for r in reqs:
                r.wait()
            top = list(range(n - NL, n))
            bot = list(range(NL))
            if lo >= 0:
                exp = _layers(U, (zb - 1) % Nz, top)
                assert np.array_equal(recv_lo.numpy(), exp), (rank, "recv_lo", p, basis, N, bc)
            else:
                assert zb == 0 and bc == "dirichlet"
            if hi >= 0:
                exp = _layers(U, ze % Nz, bot)
                assert np.array_equal(recv_hi.numpy(), exp), (rank, "recv_hi", p, basis, N, bc)
            else:
                assert ze == Nz and bc == "dirichlet"
            # partition: every plane owned exactly once, contiguous ranges
            bounds = [None] * world
            dist.all_gather_object(bounds, (zb, ze))
            assert bounds[0][0] == 0 and bounds[-1][1] == Nz
            assert all(bounds[i][1] == bounds[i + 1][0] for i in range(world - 1))
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_slab_halo_protocol(world):
    cases = [(3, "hermite", (2, 3, 5), "dirichlet"), (3, "hermite", (2, 2, 4), "periodic"),
             (5, "hermite", (3, 2, world), "periodic"), (2, "gl", (2, 2, 6), "dirichlet"),
             (1, "hermite", (2, 1, 3), "periodic")]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
    assert all(v == "ok" for _, v in res), res


def test_slab_plan_properties():
    import paper_1907_08492_b200 as P
    for Nz in (1, 5, 16, 128):
        for W in range(1, min(Nz, 8) + 1):
            for bc in ("dirichlet", "periodic"):
                plans = [P.slab_plan(Nz, W, r, bc) for r in range(W)]
                assert plans[0]["z_begin"] == 0 and plans[-1]["z_end"] == Nz
                for r in range(W):
                    pl = plans[r]
                    assert pl["z_end"] > pl["z_begin"]
                    if r < W - 1:
                        assert pl["z_end"] == plans[r + 1]["z_begin"]
                    if pl["hi_peer"] >= 0:
                        assert plans[pl["hi_peer"]]["lo_peer"] == r
                    if W == 1:
                        assert pl["lo_peer"] == pl["hi_peer"] == -1
    with pytest.raises(P.DgError):
        P.slab_plan(3, 4, 0)
