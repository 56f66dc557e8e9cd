"""CPU test of the multi-GPU host logic with world_size 2 over gloo.

Each rank takes its z-slab from the library's own partition arithmetic
(mf_partition, no GPU needed), forms its local partial result with the oracle
on the slab (the slab's cells only), applies the identity-row ownership rule
(constrained rows on a shared plane belong to the upper rank), exchanges the
shared plane's partial sums with its neighbour exactly as api.cu::halo_exchange
does (send mine, receive theirs, add) and must reproduce the global oracle
result on its slice; shared-plane copies must agree bitwise and owned-prefix
dots must sum to the global dot."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, q):
    import sys

    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import synth
        from paper_1910_13247_b200 import mf

        nc, k = case["n_cells"], case["k"]
        coeff = case.get("coeff", 1.0)
        part = mf.partition(nc, k, rank, world)
        cz0, cz1, first, n_local, n_owned, plane = (part[x] for x in
                                                    ("cz0", "cz1", "first_global", "n_local", "n_owned", "plane"))
        hz = 1.0 / nc[2]
        dirichlet = 0b001111 | (0b010000 if rank == 0 else 0) | (0b100000 if rank == world - 1 else 0)
        kw = dict(coeff_kind=1 if coeff == "variable" else 0, coeff_value=1.0 if coeff == "variable" else coeff)
        p_loc = oracle.problem(dim=3, n_cells=(nc[0], nc[1], cz1 - cz0), degree=k, lower=(0, 0, cz0 * hz),
                               upper=(1, 1, cz1 * hz), dirichlet=dirichlet, **kw)
        p_glob = oracle.problem(dim=3, n_cells=nc, degree=k, **kw)
        assert oracle.n_dofs(p_loc) == n_local
        x = synth.uniform(first, n_local, 3)  # the same values the global vector holds
        y = oracle.CSR(p_loc) @ x
        cons = oracle.constrained_mask_fast(p_loc)
        if rank < world - 1:  # identity rows on my top plane belong to the upper rank
            top = y[n_local - plane:]  # a view
            top[cons[n_local - plane:]] = 0.0
        # symmetric exchange of the shared planes (api.cu::halo_exchange)
        recv_lo = torch.zeros(plane, dtype=torch.float64)
        recv_hi = torch.zeros(plane, dtype=torch.float64)
        reqs = []
        if rank < world - 1:
            reqs.append(dist.isend(torch.from_numpy(y[n_local - plane:].copy()), rank + 1))
            reqs.append(dist.irecv(recv_hi, rank + 1))
        if rank > 0:
            reqs.append(dist.isend(torch.from_numpy(y[:plane].copy()), rank - 1))
            reqs.append(dist.irecv(recv_lo, rank - 1))
        for r in reqs:
            r.wait()
        if rank < world - 1:
            y[n_local - plane:] = y[n_local - plane:] + recv_hi.numpy()
        if rank > 0:
            y[:plane] = y[:plane] + recv_lo.numpy()
        y_ref = (oracle.CSR(p_glob) @ synth.uniform(0, oracle.n_dofs(p_glob), 3))[first:first + n_local]
        err = np.linalg.norm(y - y_ref) / np.linalg.norm(y_ref)
        # bitwise agreement of the two copies of each shared plane
        same = True
        if rank < world - 1:
            dist.send(torch.from_numpy(y[n_local - plane:].copy()), rank + 1)
        if rank > 0:
            other = torch.zeros(plane, dtype=torch.float64)
            dist.recv(other, rank - 1)
            same = bool(np.array_equal(other.numpy(), y[:plane]))
        # owned-prefix dot summed over ranks == global dot
        d = torch.tensor([float(x[:n_owned] @ y[:n_owned])], dtype=torch.float64)
        dist.all_reduce(d)
        xg = synth.uniform(0, oracle.n_dofs(p_glob), 3)
        yg = oracle.CSR(p_glob) @ xg
        dot_err = abs(d.item() - float(xg @ yg)) / abs(float(xg @ yg))
        q.put((rank, err, same, dot_err))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", [
    dict(n_cells=(3, 4, 5), k=2),
    dict(n_cells=(2, 3, 4), k=3, coeff="variable"),
    dict(n_cells=(3, 2, 2), k=4, coeff=2.0),
])
def test_zslab_exchange_reproduces_global_operator(case):
    from paper_1910_13247_b200 import build

    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    res = sorted(q.get(timeout=10) for _ in range(2))
    for rank, err, same, dot_err in res:
        assert err <= 1e-13, (rank, err)
        assert same, rank
        assert dot_err <= 1e-12, (rank, dot_err)
    assert all(p.exitcode == 0 for p in procs)


def test_partition_arithmetic():
    from paper_1910_13247_b200 import build, mf

    build.build()
    nc, k = (7, 5, 11), 3
    N = [k * n + 1 for n in nc]
    for world in (1, 2, 3, 4, 8, 11):
        parts = [mf.partition(nc, k, r, world) for r in range(world)]
        assert parts[0]["cz0"] == 0 and parts[-1]["cz1"] == nc[2]
        for a, b in zip(parts, parts[1:]):
            assert a["cz1"] == b["cz0"]
            # the shared plane: last plane of a == first plane of b
            assert a["first_global"] + a["n_local"] - a["plane"] == b["first_global"]
        assert sum(p["n_owned"] for p in parts) == N[0] * N[1] * N[2]
        for p in parts:
            assert p["plane"] == N[0] * N[1]
            assert p["n_local"] == p["plane"] * (k * (p["cz1"] - p["cz0"]) + 1)
    with pytest.raises(mf.MFError):
        mf.partition(nc, k, 0, 12)  # fewer z layers than ranks
