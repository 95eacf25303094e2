"""Column-sharded PSCA protocol (large.ShardedDriver) over gloo, world_size 2, on CPU.

The GPU stepper (large.GpuLargeStepper) exchanges, per iteration, one
contiguous block [rank-local Sigma increment | sum dx^2 | prior partial]
(sum) and min q (min).  Here a
numpy stepper with the same step semantics -- incremental D_{k+1} =
(1-rho_k) D_k + S diag(rho cand g) S^H, replicated factorisation, local
column updates -- runs on each rank's block of columns and the driver's
all-reduces go through gloo.  The assembled result must equal the
single-process oracle (which recomputes Sigma from scratch each iteration).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import psca_oracle as orc   # checker / test stepper only


class NumpyStepper:
    """Test double of GpuLargeStepper: same begin/columns/exchange/factor protocol."""

    def __init__(self, kind, S, g, E, noise, M, steps, max_iter, tol=0.0):
        self.kind, self.S, self.g, self.E, self.noise = kind, S, g, E, noise
        self.M, self.steps, self.T, self.tol = M, steps, max_iter, tol
        self.L, self.N = S.shape
        self.known = kind in ("ml-k", "map-k")

    def _factor(self, sigma):
        self.frob = np.linalg.norm(sigma)
        self.P = orc.herm_inverse(sigma)
        self.A = self.P @ self.E @ self.P

    def begin(self):
        self.x = np.zeros(self.N)
        self.D = np.zeros((self.L, self.L), complex)
        self.status, self.n_iter, self.stop = 0, 0, False
        self.update_norm = []
        self._factor(self.D + self.noise * np.eye(self.L))

    def columns(self, k):
        if self.stop:            # gated like the device kernels after a stop
            return
        q, r = orc.quad(self.S, self.P, self.E)
        d = q - r
        grad = self.g * d if self.known else d
        coef = (self.g * q) ** 2 if self.known else q ** 2
        hi = 1.0 if self.known else np.inf
        cand = np.clip(self.x - grad / coef, 0.0, hi)
        rho = self.steps[k]
        rc = rho * cand
        self.x_next = (1.0 - rho) * self.x + rc
        v = rc * self.g if self.known else rc
        inc = (self.S * v) @ self.S.conj().T
        dx2 = float(np.sum((self.x_next - self.x) ** 2))
        self._sum = torch.from_numpy(np.concatenate([np.ascontiguousarray(inc).view(np.float64).ravel(),
                                                     [dx2, 0.0]]))
        self._minq = torch.tensor([float(np.min(q)) if q.size else np.inf], dtype=torch.float64)

    def exchange(self):
        return self._sum, self._minq

    def factor(self, k):
        if self.stop:
            return
        if float(self._minq[0]) < 0.5 * self.L / self.frob:
            self.status, self.stop = 2, True
            return
        un = np.sqrt(float(self._sum[-2]))
        self.update_norm.append(un)
        self.x = self.x_next
        self.n_iter = k + 1
        if un < self.tol or k + 1 >= self.T:
            self.stop = True
            return
        inc = self._sum[:-2].numpy().view(np.complex128).reshape(self.L, self.L)
        self.D = (1.0 - self.steps[k]) * self.D + inc
        self._factor(self.D + self.noise * np.eye(self.L))

    def stopped(self):
        return self.stop

    def result(self):
        return {"x": self.x, "update_norm": np.array(self.update_norm), "status": self.status,
                "n_iter": self.n_iter}


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, inputs, out_q, tol=0.0):
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    from paper_2503_15259_b200.large import ShardedDriver, column_shard
    kind, S, g, E, M, steps, T = inputs
    sl = column_shard(S.shape[1], rank, world)
    st = NumpyStepper(kind, S[:, sl], g[sl], E, 1.0, M, steps, T, tol=tol)
    res = ShardedDriver(st, group=dist.group.WORLD, dist=dist).run(T)
    out_q.put((rank, res["x"], res["update_norm"], res["n_iter"]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("kind,tol", [("ml-k", 0.0), ("ml-ud", 0.0), ("ml-ud", 50.0)])
def test_two_rank_column_sharding_matches_single_process(kind, tol):
    """tol > 0: an early stop, seen by the driver at its next flag check (every 8
    iterations); the gated steppers keep the stopped state."""
    from paper_2503_15259_b200 import scenes
    cfg = scenes.SceneConfig(13, kind, 301, 24, 64, 20, 25, 1)
    s = scenes.make_scene(cfg, 0)
    T = 25
    steps = orc.default_steps(T)
    inputs = (kind, s.pilots, s.gains, s.emp_cov, 64, steps, T)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, inputs, q, tol)) for r in range(2)]
    for p in procs:
        p.start()
    outs = sorted([q.get(timeout=300) for _ in range(2)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    x = np.concatenate([o[1] for o in outs])
    ref = orc.psca(kind, s.pilots, s.gains, s.emp_cov, 1.0, 64, steps, T, tol=tol)
    assert outs[0][3] == outs[1][3] == len(ref["update_norm"])
    if tol > 0:
        assert outs[0][3] < T
    np.testing.assert_allclose(outs[0][2], outs[1][2], rtol=0, atol=0)   # replicated scalars
    assert np.max(np.abs(x - ref["final"])) <= 1e-9 * np.max(np.abs(ref["final"]))
    assert np.max(np.abs(outs[0][2] - ref["update_norm"])) <= 1e-9 * np.max(ref["update_norm"])


def test_column_shard_partition():
    from paper_2503_15259_b200.large import column_shard
    for n, w in ((100_000, 8), (1000, 3), (7, 4)):
        parts = [column_shard(n, r, w) for r in range(w)]
        cover = np.concatenate([np.arange(n)[p] for p in parts])
        np.testing.assert_array_equal(cover, np.arange(n))
