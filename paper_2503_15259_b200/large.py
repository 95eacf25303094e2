"""Large pilot length path (L <= 256) and multi-GPU column sharding of one instance.

BASELINE config 4 (N = 100,000 devices, L = 256, one instance) runs here: the
PSCA loop (estimators.py:259-286) becomes a host-driven step loop over the
C ABI ``psca_large_*`` entry points (csrc/psca_large.cuh):

    stepper.begin()                       x = 0, Sigma_0 = sigma^2 I, factor
    for k in range(T):
        stepper.columns(k)                this rank's columns: quad forms, update,
                                          partial Sigma increment, dx2, prior, min q
        all_reduce([increment | dx2 | prior], SUM); all_reduce(min q, MIN)
        stepper.factor(k)                 finalise k, factor Sigma_{k+1}
        every 8 iterations: if stepper.stopped(): break

With ``group=None`` (one GPU) the all-reduces are skipped.  With a
torch.distributed process group (NCCL, one process per GPU) each rank holds
a contiguous block of columns (devices) of the one instance; the exchange is
ONE sum all-reduce of a contiguous block -- the L x L partial increment
(about 0.5 MiB at L = 256 in C-fragment form), sum dx^2 and the shard's prior
penalty -- and one min all-reduce of min q per iteration.  The factorisation
is replicated, so every rank holds identical P'/A' fragments.  Every kernel of
the step is gated on the device stop flag, so the loop checks the flag on the
host only every ``check_every`` iterations (no per-iteration synchronisation).

``ShardedDriver`` only talks to a stepper object; tests drive it with a numpy
stepper over gloo (tests/test_sharded_cpu.py) to check the protocol.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import device
from .device import EffPriorC, PscaNativeError


class LargeArgsC(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int), ("N", ctypes.c_int), ("L", ctypes.c_int),
        ("n_antennas", ctypes.c_int), ("max_iter", ctypes.c_int),
        ("record_objective", ctypes.c_int), ("tol", ctypes.c_double),
        ("noise", ctypes.c_double),
        ("pilots", ctypes.c_void_p), ("gains", ctypes.c_void_p), ("emp_cov", ctypes.c_void_p),
        ("steps", ctypes.c_void_p), ("prior_lin", ctypes.c_void_p), ("prior_p", ctypes.c_void_p),
        ("eff", EffPriorC),
        ("x_a", ctypes.c_void_p), ("x_b", ctypes.c_void_p), ("update_norm", ctypes.c_void_p),
        ("objective", ctypes.c_void_p), ("iterates", ctypes.c_void_p),
        ("status", ctypes.c_void_p), ("n_iter", ctypes.c_void_p), ("cond_est", ctypes.c_void_p),
        ("prior_c1", ctypes.c_void_p), ("prior_c2_indptr", ctypes.c_void_p),
        ("prior_c2_indices", ctypes.c_void_p), ("prior_c2_data", ctypes.c_void_p),
    ]


_SIGS = {
    "psca_large_workspace_bytes": (ctypes.c_size_t, [ctypes.POINTER(LargeArgsC)]),
    "psca_large_exchange": (ctypes.c_int, [ctypes.POINTER(LargeArgsC), ctypes.c_void_p,
                                           ctypes.POINTER(ctypes.c_void_p),
                                           ctypes.POINTER(ctypes.c_size_t),
                                           ctypes.POINTER(ctypes.c_void_p)]),
    "psca_large_flag": (ctypes.c_int, [ctypes.POINTER(LargeArgsC), ctypes.c_void_p,
                                       ctypes.c_void_p]),
    "psca_large_begin": (ctypes.c_int, [ctypes.POINTER(LargeArgsC), ctypes.c_void_p,
                                        ctypes.c_size_t, ctypes.c_void_p]),
    "psca_large_columns": (ctypes.c_int, [ctypes.POINTER(LargeArgsC), ctypes.c_int,
                                          ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "psca_large_factor": (ctypes.c_int, [ctypes.POINTER(LargeArgsC), ctypes.c_int,
                                         ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
}
EXPORTED_SYMBOLS = tuple(_SIGS)


def _lib():
    lib = device.load()
    if not getattr(lib, "_large_bound", False):
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        lib._large_bound = True
    return lib


class GpuLargeStepper:
    """One rank's share (a block of columns) of one large-L instance on the GPU."""

    def __init__(self, kind, pilots, gains, emp_cov, noise, n_antennas, steps, *, max_iter,
                 tol=0.0, prior_lin=None, prior_p=None, eff_prior=None,
                 record_objective=False, record_iterates=False, prior_c1=None, prior_c2=None):
        torch = device._torch()
        self.torch = torch
        self.lib = _lib()
        dev = torch.device("cuda", torch.cuda.current_device())
        f64, c128 = torch.float64, torch.complex128
        self.S = device._dev(torch, pilots, c128, dev)
        L, N = self.S.shape
        self.L, self.N, self.T = L, N, int(max_iter)
        self.E = device._dev(torch, emp_cov, c128, dev).reshape(L, L)
        self.g = device._dev(torch, gains, f64, dev).reshape(N) if gains is not None else None
        self.steps = device._dev(torch, steps, f64, dev).reshape(-1)
        self.pl = device._dev(torch, prior_lin, f64, dev) if prior_lin is not None else None
        self.pp = device._dev(torch, prior_p, f64, dev) if prior_p is not None else None
        # pairwise MVB prior (priors.py:56-159): c1 and the CSR interaction matrix
        self.c1 = self.c2p = self.c2i = self.c2d = None
        if prior_c1 is not None or prior_c2 is not None:
            if prior_c1 is None or prior_c2 is None:
                raise ValueError("the pairwise prior needs both prior_c1 and prior_c2")
            indptr, indices, data = prior_c2
            self.c1 = device._dev(torch, np.broadcast_to(np.asarray(prior_c1, dtype=float), (N,)).copy(),
                                  f64, dev)
            self.c2p = device._dev(torch, np.asarray(indptr, dtype=np.int32), torch.int32, dev)
            self.c2i = device._dev(torch, np.asarray(indices, dtype=np.int32), torch.int32, dev)
            self.c2d = device._dev(torch, np.asarray(data, dtype=float), f64, dev)
            if self.c2p.numel() != N + 1:
                raise ValueError("prior_c2 indptr must have N + 1 entries")
        T = max(self.T, 1)
        self.x_a = torch.empty(N, dtype=f64, device=dev)
        self.x_b = torch.empty(N, dtype=f64, device=dev)
        self.un = torch.empty(T, dtype=f64, device=dev)
        self.obj = torch.zeros(T, dtype=f64, device=dev) if record_objective else None
        self.its = torch.zeros((self.T + 1, N), dtype=f64, device=dev) if record_iterates else None
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        self.n_iter = torch.zeros(1, dtype=torch.int32, device=dev)
        self.cond = torch.zeros(1, dtype=f64, device=dev)
        ptr = lambda t: t.data_ptr() if t is not None else 0   # noqa: E731
        self.args = LargeArgsC(
            kind=device.KIND_CODES[kind], N=N, L=L, n_antennas=int(n_antennas),
            max_iter=self.T, record_objective=int(bool(record_objective)), tol=float(tol),
            noise=float(noise), pilots=ptr(self.S), gains=ptr(self.g), emp_cov=ptr(self.E),
            steps=ptr(self.steps), prior_lin=ptr(self.pl), prior_p=ptr(self.pp),
            eff=device.eff_prior_struct(eff_prior), x_a=ptr(self.x_a), x_b=ptr(self.x_b),
            update_norm=ptr(self.un), objective=ptr(self.obj), iterates=ptr(self.its),
            status=ptr(self.status), n_iter=ptr(self.n_iter), cond_est=ptr(self.cond),
            prior_c1=ptr(self.c1), prior_c2_indptr=ptr(self.c2p), prior_c2_indices=ptr(self.c2i),
            prior_c2_data=ptr(self.c2d))
        nbytes = self.lib.psca_large_workspace_bytes(ctypes.byref(self.args))
        if nbytes == 0:
            raise PscaNativeError("psca_large rejected the arguments (shape/kind/pointers)")
        self.ws = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        dsig, n, red = ctypes.c_void_p(), ctypes.c_size_t(), ctypes.c_void_p()
        device._check(self.lib.psca_large_exchange(ctypes.byref(self.args), self._ws(),
                                                   ctypes.byref(dsig), ctypes.byref(n),
                                                   ctypes.byref(red)), "psca_large_exchange")
        base = self.ws.data_ptr()
        assert red.value == dsig.value + 8 * n.value, "exchange block must be contiguous"
        self.xsum = self.ws[dsig.value - base: dsig.value - base + 8 * (n.value + 2)].view(f64)
        self.dsig = self.xsum[:n.value]
        self.red = self.ws[red.value - base: red.value - base + 32].view(f64)
        fp = ctypes.c_void_p()
        device._check(self.lib.psca_large_flag(ctypes.byref(self.args), self._ws(),
                                               ctypes.byref(fp)), "psca_large_flag")
        self.flag = self.ws[fp.value - base: fp.value - base + 4].view(torch.int32)
        self.launches = 0

    def _ws(self):
        return ctypes.c_void_p(self.ws.data_ptr())

    def _call(self, name, *k):
        fn = getattr(self.lib, name)
        device._check(fn(ctypes.byref(self.args), *k, self._ws(),
                         ctypes.c_size_t(self.ws.numel()), device._stream(self.torch)), name)
        self.launches += self.lib.psca_last_launch_count()

    def begin(self):
        self._call("psca_large_begin")

    def columns(self, k):
        self._call("psca_large_columns", ctypes.c_int(k))

    def factor(self, k):
        self._call("psca_large_factor", ctypes.c_int(k))

    def exchange(self):
        """(sum-reduced block [increment | dx2 | prior], min-reduced [min q]) views."""
        return self.xsum, self.red[2:3]

    def stopped(self) -> bool:
        return bool(self.flag.item())

    def result(self) -> dict:
        status = int(self.status.item())
        k_done = int(self.n_iter.item())
        # x after k iterations lives in x_a for even k, x_b for odd k
        x = self.x_a if k_done % 2 == 0 else self.x_b
        return {"x": x.clone(), "update_norm": self.un[:k_done].clone(), "status": status,
                "n_iter": k_done, "cond_est": float(self.cond.item()),
                "objective": self.obj[:k_done].clone() if self.obj is not None else None,
                "iterates": self.its[:k_done + 1].clone() if self.its is not None else None}


class ShardedDriver:
    """PSCA step loop with optional column sharding over a process group."""

    def __init__(self, stepper, group=None, dist=None, check_every: int = 8):
        self.stepper = stepper
        self.group = group
        self.dist = dist
        self.check_every = max(1, int(check_every))
        if group is not None and dist is None:
            import torch.distributed as dist_mod
            self.dist = dist_mod

    def run(self, max_iter: int) -> dict:
        st = self.stepper
        st.begin()
        for k in range(max_iter):
            st.columns(k)
            if self.group is not None:
                xsum, minq = st.exchange()
                d = self.dist
                d.all_reduce(xsum, op=d.ReduceOp.SUM, group=self.group)
                d.all_reduce(minq, op=d.ReduceOp.MIN, group=self.group)
            st.factor(k)
            # the stop flag is replicated on every rank (it follows from reduced
            # values), so all ranks leave at the same k
            if (k + 1) % self.check_every == 0 and k + 1 < max_iter and st.stopped():
                break
        return st.result()


def column_shard(n_devices: int, rank: int, world: int) -> slice:
    """Contiguous block of devices (columns) owned by ``rank``."""
    per = (n_devices + world - 1) // world
    lo = min(n_devices, rank * per)
    return slice(lo, min(n_devices, lo + per))


def psca_run_large(kind, pilots, gains, emp_cov, noise, n_antennas, steps, *, max_iter, tol=0.0,
                   prior_lin=None, prior_p=None, eff_prior=None, record_objective=False,
                   record_iterates=False, group=None, prior_c1=None, prior_c2=None) -> dict:
    """Solve one instance with the large-L step loop (columns = this rank's shard)."""
    if prior_c1 is not None and group is not None and group.size() > 1:
        # the row sums c2 x couple devices of different shards (an all-gather of x
        # per iteration would be needed); the reference's group priors are small-N
        raise NotImplementedError("pairwise MAP-K prior with column shards")
    st = GpuLargeStepper(kind, pilots, gains, emp_cov, noise, n_antennas, steps,
                         max_iter=max_iter, tol=tol, prior_lin=prior_lin, prior_p=prior_p,
                         eff_prior=eff_prior, record_objective=record_objective,
                         record_iterates=record_iterates, prior_c1=prior_c1, prior_c2=prior_c2)
    res = ShardedDriver(st, group=group).run(max_iter)
    res["launches"] = st.launches
    return res
