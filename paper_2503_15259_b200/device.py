"""ctypes binding of the C ABI in include/psca.h (the product's only compute path).

torch is used for device memory, streams and host<->device copies only; every
FLOP of the solver runs in ``_psca.so`` (built from ``csrc/psca.cu`` for
sm_100a).  There is no CPU fallback: a missing library or a missing GPU raises.
"""

from __future__ import annotations

import ctypes
import math
import pathlib
import threading

import numpy as np

_HERE = pathlib.Path(__file__).resolve().parent
LIB_PATH = _HERE / "_psca.so"

KIND_CODES = {"ml-k": 0, "map-k": 1, "ml-ud": 2, "map-ur": 3}
STATUS_RUNNING, STATUS_CHOL_FAIL, STATUS_QFLOOR, STATUS_CONVERGED = 0, 1, 2, 3

_lock = threading.Lock()
_lib = None


class PscaNativeError(RuntimeError):
    """The CUDA library is missing, the GPU is missing, or a call failed."""


class EffPriorC(ctypes.Structure):
    _fields_ = [(name, ctypes.c_double) for name in
                ("eps", "g_low", "g_high", "dead_zone_grad", "p_lin", "k", "eta", "area2",
                 "cv", "cw")]


class SolveArgsC(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int), ("B", ctypes.c_int), ("N", ctypes.c_int), ("L", ctypes.c_int),
        ("n_antennas", ctypes.c_int), ("max_iter", ctypes.c_int), ("tol", ctypes.c_double),
        ("record_objective", ctypes.c_int), ("n_chunks", ctypes.c_int),
        ("pilots", ctypes.c_void_p), ("gains", ctypes.c_void_p), ("emp_cov", ctypes.c_void_p),
        ("noise", ctypes.c_void_p), ("steps", ctypes.c_void_p), ("prior_lin", ctypes.c_void_p),
        ("prior_p", ctypes.c_void_p), ("eff", EffPriorC),
        ("prior_c1", ctypes.c_void_p), ("prior_c2_indptr", ctypes.c_void_p),
        ("prior_c2_indices", ctypes.c_void_p), ("prior_c2_data", ctypes.c_void_p),
        ("x_out", ctypes.c_void_p), ("update_norm", ctypes.c_void_p),
        ("objective", ctypes.c_void_p), ("iterates", ctypes.c_void_p),
        ("status", ctypes.c_void_p), ("n_iter", ctypes.c_void_p), ("cond_est", ctypes.c_void_p),
        ("fault_iter", ctypes.c_int),
        ("steps_stride", ctypes.c_int),
    ]


class PriorArgsC(ctypes.Structure):
    """psca_prior_args (include/psca.h)."""
    _fields_ = [
        ("kind", ctypes.c_int), ("B", ctypes.c_int), ("N", ctypes.c_int),
        ("n_antennas", ctypes.c_int), ("x", ctypes.c_void_p), ("prior_lin", ctypes.c_void_p),
        ("prior_p", ctypes.c_void_p), ("eff", EffPriorC), ("prior_c1", ctypes.c_void_p),
        ("prior_c2_indptr", ctypes.c_void_p), ("prior_c2_indices", ctypes.c_void_p),
        ("prior_c2_data", ctypes.c_void_p), ("grad", ctypes.c_void_p),
        ("value", ctypes.c_void_p), ("density", ctypes.c_void_p),
    ]


class CoordArgsC(ctypes.Structure):
    """psca_coord_args (include/psca.h)."""
    _fields_ = [
        ("kind", ctypes.c_int), ("B", ctypes.c_int), ("N", ctypes.c_int), ("L", ctypes.c_int),
        ("rho", ctypes.c_double), ("hi", ctypes.c_double),
        ("x", ctypes.c_void_p), ("q", ctypes.c_void_p), ("r", ctypes.c_void_p),
        ("gains", ctypes.c_void_p), ("prior_grad", ctypes.c_void_p), ("sigma", ctypes.c_void_p),
        ("grad", ctypes.c_void_p), ("coef", ctypes.c_void_p), ("cand", ctypes.c_void_p),
        ("x_new", ctypes.c_void_p), ("update_norm", ctypes.c_void_p), ("status", ctypes.c_void_p),
    ]


# exported symbols and their signatures (must match include/psca.h)
class BcdArgsC(ctypes.Structure):
    """psca_bcd_args (include/psca.h)."""
    _fields_ = [
        ("kind", ctypes.c_int), ("B", ctypes.c_int), ("N", ctypes.c_int), ("L", ctypes.c_int),
        ("n_antennas", ctypes.c_int), ("init", ctypes.c_int),
        ("pilots", ctypes.c_void_p), ("gains", ctypes.c_void_p), ("emp_cov", ctypes.c_void_p),
        ("noise", ctypes.c_void_p), ("prior_lin", ctypes.c_void_p), ("prior_c1", ctypes.c_void_p),
        ("prior_c2_indptr", ctypes.c_void_p), ("prior_c2_indices", ctypes.c_void_p),
        ("prior_c2_data", ctypes.c_void_p), ("x", ctypes.c_void_p), ("sigma_inv", ctypes.c_void_p),
        ("status", ctypes.c_void_p),
    ]


_SIGS = {
    "psca_version": (ctypes.c_char_p, []),
    "psca_last_error": (ctypes.c_char_p, []),
    "psca_last_launch_count": (ctypes.c_int, []),
    "psca_last_path": (ctypes.c_int, []),
    "psca_profile_begin": (ctypes.c_int, []),
    "psca_profile_end": (ctypes.c_int, [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int),
                                        ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int)]),
    "psca_set_serial": (ctypes.c_int, [ctypes.c_int]),
    "psca_debug_probes": (ctypes.c_int, [ctypes.POINTER(ctypes.c_longlong), ctypes.c_int]),
    "psca_profile_launches": (ctypes.c_int, [ctypes.POINTER(ctypes.c_double),
                                             ctypes.POINTER(ctypes.c_int), ctypes.c_int]),
    "psca_solve_workspace_bytes": (ctypes.c_size_t, [ctypes.POINTER(SolveArgsC)]),
    "psca_solve": (ctypes.c_int, [ctypes.POINTER(SolveArgsC), ctypes.c_void_p, ctypes.c_size_t,
                                  ctypes.c_void_p]),
    "psca_empirical_cov": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                          ctypes.c_void_p]),
    "psca_received": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                     ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                     ctypes.c_void_p]),
    "psca_cov_workspace_bytes": (ctypes.c_size_t, [ctypes.c_int, ctypes.c_int, ctypes.c_int]),
    "psca_cov_unknown": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                        ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "psca_inverse_workspace_bytes": (ctypes.c_size_t, [ctypes.c_int, ctypes.c_int]),
    "psca_hpd_inverse": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                        ctypes.c_void_p]),
    "psca_quad_workspace_bytes": (ctypes.c_size_t, [ctypes.c_int, ctypes.c_int, ctypes.c_int]),
    "psca_quad_forms": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                       ctypes.c_void_p]),
    "psca_bcd_sweep": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    "psca_prior_terms": (ctypes.c_int, [ctypes.POINTER(PriorArgsC), ctypes.c_void_p]),
    "psca_coord_step": (ctypes.c_int, [ctypes.POINTER(CoordArgsC), ctypes.c_void_p]),
    "psca_objective_workspace_bytes": (ctypes.c_size_t, [ctypes.c_int, ctypes.c_int]),
    "psca_eval_objective": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                           ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                           ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                           ctypes.c_void_p]),
}
EXPORTED_SYMBOLS = tuple(_SIGS)


def load() -> ctypes.CDLL:
    """Load ``_psca.so`` (raises PscaNativeError when it has not been built)."""
    global _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise PscaNativeError(
                    f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                    "g.build()'` (there is no CPU fallback)")
            lib = ctypes.CDLL(str(LIB_PATH))
            for name, (res, args) in _SIGS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise PscaNativeError("the PSCA solver needs a CUDA GPU (sm_100a); none is visible")
    return torch


def _check(rc: int, what: str):
    if rc != 0:
        names = {-1: "bad argument", -2: "CUDA error", -3: "workspace too small",
                 -4: "unsupported shape"}
        detail = ""
        if rc == -2 and _lib is not None:
            detail = f" ({_lib.psca_last_error().decode()})"
        raise PscaNativeError(f"{what} failed: {names.get(rc, rc)}{detail}")


def _stream(torch):
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def _workspace(torch, nbytes: int, device):
    return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=device)


def _dev(torch, arr, dtype, device):
    if isinstance(arr, torch.Tensor):
        return arr.to(device=device, dtype=dtype).contiguous()
    return torch.as_tensor(np.ascontiguousarray(arr), dtype=dtype, device=device)


# ---------------------------------------------------------------------------
# the batched solver (device tensors in, device tensors out)
# ---------------------------------------------------------------------------

def eff_prior_struct(prior) -> EffPriorC:
    """psca_eff_prior from an EffPathlossPrior-like object (priors.py:173-281)."""
    if prior is None:
        return EffPriorC()
    p_lin = 10.0 ** (prior.tx_power_dbm / 10.0)
    k = 4.0 * np.pi / prior.wavelength
    cv, cw = prior._hermite_coeffs()
    return EffPriorC(eps=float(prior.eps), g_low=float(prior.g_low), g_high=float(prior.g_high),
                     dead_zone_grad=float(prior.dead_zone_grad), p_lin=float(p_lin), k=float(k),
                     eta=float(prior.pathloss_exp),
                     area2=float(prior.d_outer ** 2 - prior.d_inner ** 2), cv=float(cv),
                     cw=float(cw))


def solve(kind: str, pilots, emp_cov, noise, n_antennas: int, steps, *, gains=None,
          prior_lin=None, prior_p=None, eff_prior=None, prior_c1=None, prior_c2=None,
          max_iter: int | None = None, tol: float = 0.0, record_objective: bool = False,
          record_iterates: bool = False, n_chunks: int = 0, out=None, fault_iter: int = 0):
    """Run the batched PSCA solve on the current CUDA device / stream.

    pilots (B,L,N) complex128, emp_cov (B,L,L) complex128, noise (B,) float64,
    gains (B,N) float64 for known-pathloss kinds, steps (T,) float64 (one
    schedule for the batch) or (B, T) (one schedule per instance).
    A pairwise MAP-K prior passes prior_c1 (N,) and prior_c2 = (indptr,
    indices, data) of its CSR interaction matrix instead of prior_lin.
    Inputs may be numpy arrays or torch tensors (moved to the device if
    needed).  Returns a dict of device tensors: x (B,N), update_norm (B,T),
    objective (B,T) or None, iterates (B,T+1,N) or None, status (B,) int32,
    n_iter (B,) int32, cond_est (B,).  ``fault_iter`` = k >= 1 forces the
    factorisation opening iteration k-1 to fail (the test seam of psca.h).
    """
    torch = _torch()
    lib = load()
    dev = torch.device("cuda", torch.cuda.current_device())
    if kind not in KIND_CODES:
        raise ValueError(f"unknown problem kind {kind!r}")
    S = _dev(torch, pilots, torch.complex128, dev)
    if S.dim() != 3:
        raise ValueError("pilots must be (B, L, N)")
    B, L, N = S.shape
    E = _dev(torch, emp_cov, torch.complex128, dev)
    sig2 = _dev(torch, noise, torch.float64, dev).reshape(B)
    st = _dev(torch, steps, torch.float64, dev)
    stride = 0
    if st.dim() == 2:
        if st.shape[0] != B:
            raise ValueError("per-instance steps must be (B, T)")
        st = st.contiguous()
        stride = int(st.shape[1])
    st = st.reshape(-1)
    T = (stride or int(st.numel())) if max_iter is None else int(max_iter)
    if (stride or st.numel()) < T:
        raise ValueError("need one step per iteration")
    g = _dev(torch, gains, torch.float64, dev) if gains is not None else None
    pl = _dev(torch, prior_lin, torch.float64, dev) if prior_lin is not None else None
    pp = _dev(torch, prior_p, torch.float64, dev) if prior_p is not None else None
    c1 = _dev(torch, prior_c1, torch.float64, dev) if prior_c1 is not None else None
    c2 = None
    if prior_c2 is not None:
        indptr, indices, data = prior_c2
        c2 = (_dev(torch, np.asarray(indptr, dtype=np.int32), torch.int32, dev),
              _dev(torch, np.asarray(indices, dtype=np.int32), torch.int32, dev),
              _dev(torch, np.asarray(data, dtype=np.float64), torch.float64, dev))
        if c2[1].numel() == 0:   # keep valid pointers for an empty interaction
            c2 = (c2[0], torch.zeros(1, dtype=torch.int32, device=dev),
                  torch.zeros(1, dtype=torch.float64, device=dev))
    if out is None:
        out = {}
    # output buffers are reused from ``out`` when the shapes match, so repeated
    # solves with the same inputs present identical arguments to psca_solve
    # (whose CUDA-graph cache then replays the launch sequence)
    bufs = out.get("_bufs") or {}

    def buf(name, shape, dtype):
        t = bufs.get(name)
        if t is None or tuple(t.shape) != tuple(shape) or t.dtype != dtype or t.device != dev:
            t = torch.empty(shape, dtype=dtype, device=dev)
            bufs[name] = t
        return t

    x = out.get("x")
    if x is None or tuple(x.shape) != (B, N) or x.device != dev:
        x = torch.empty((B, N), dtype=torch.float64, device=dev)
    un = buf("un", (B, max(T, 1)), torch.float64)
    obj = buf("obj", (B, max(T, 1)), torch.float64) if record_objective else None
    its = buf("its", (B, T + 1, N), torch.float64) if record_iterates else None
    status = buf("status", (B,), torch.int32)
    n_iter = buf("n_iter", (B,), torch.int32)
    cond = buf("cond", (B,), torch.float64)
    args = SolveArgsC(
        kind=KIND_CODES[kind], B=B, N=N, L=L, n_antennas=int(n_antennas), max_iter=T,
        tol=float(tol), record_objective=int(bool(record_objective)), n_chunks=int(n_chunks),
        pilots=S.data_ptr(), gains=g.data_ptr() if g is not None else 0, emp_cov=E.data_ptr(),
        noise=sig2.data_ptr(), steps=st.data_ptr(),
        prior_lin=pl.data_ptr() if pl is not None else 0,
        prior_p=pp.data_ptr() if pp is not None else 0,
        eff=eff_prior_struct(eff_prior),
        prior_c1=c1.data_ptr() if c1 is not None else 0,
        prior_c2_indptr=c2[0].data_ptr() if c2 is not None else 0,
        prior_c2_indices=c2[1].data_ptr() if c2 is not None else 0,
        prior_c2_data=c2[2].data_ptr() if c2 is not None else 0,
        x_out=x.data_ptr(), update_norm=un.data_ptr(),
        objective=obj.data_ptr() if obj is not None else 0,
        iterates=its.data_ptr() if its is not None else 0, status=status.data_ptr(),
        n_iter=n_iter.data_ptr(), cond_est=cond.data_ptr(), fault_iter=int(fault_iter),
        steps_stride=stride)
    nbytes = lib.psca_solve_workspace_bytes(ctypes.byref(args))
    if nbytes == 0 and B > 0:
        raise PscaNativeError("psca_solve rejected the arguments (shape/kind/pointers)")
    ws = out.get("_ws")
    if ws is None or ws.numel() < nbytes:
        ws = _workspace(torch, nbytes, dev)
    _check(lib.psca_solve(ctypes.byref(args), _ptr(ws), ctypes.c_size_t(ws.numel()),
                          _stream(torch)), "psca_solve")
    return {"x": x, "update_norm": un[:, :T], "objective": obj[:, :T] if obj is not None else None,
            "iterates": its, "status": status, "n_iter": n_iter, "cond_est": cond, "_ws": ws,
            "_bufs": bufs,
            "launches": lib.psca_last_launch_count(),
            "path": {0: "two-kernel", 1: "persistent", 2: "two-kernel-split"}.get(
                lib.psca_last_path(), "?")}


# ---------------------------------------------------------------------------
# component entry points (numpy or tensors in; numpy out for numpy input)
# ---------------------------------------------------------------------------

def _batched(arr, ndim):
    a = np.asarray(arr)
    return (a[None], True) if a.ndim == ndim else (a, False)


def empirical_cov(y, n_antennas: int):
    torch = _torch()
    lib = load()
    ya, single = _batched(y, 2)
    dev = torch.device("cuda", torch.cuda.current_device())
    Y = _dev(torch, ya, torch.complex128, dev)
    B, L, Mc = Y.shape
    out = torch.empty((B, L, L), dtype=torch.complex128, device=dev)
    _check(lib.psca_empirical_cov(_ptr(Y), B, L, Mc, int(n_antennas), _ptr(out), _stream(torch)),
           "psca_empirical_cov")
    res = out.cpu().numpy()
    return res[0] if single else res


def received_t(S, active, gains, H, Z):
    """Y = S[:, active] diag(sqrt(g[active])) H + Z on the device (psca_received).

    S (B,L,N) c128, active (B,K) int, gains (B,N), H (B,K,M) c128, Z (B,L,M) c128,
    all CUDA tensors (converted / made contiguous here); returns Y (B,L,M)."""
    torch = _torch()
    lib = load()
    dev = S.device
    S = S.to(torch.complex128).contiguous()
    A = active.to(device=dev, dtype=torch.int32).contiguous()
    g = gains.to(device=dev, dtype=torch.float64).contiguous()
    H = H.to(device=dev, dtype=torch.complex128).contiguous()
    Z = Z.to(device=dev, dtype=torch.complex128).contiguous()
    B, L, N = S.shape
    K, M = H.shape[1], H.shape[2]
    Y = torch.empty((B, L, M), dtype=torch.complex128, device=dev)
    _check(lib.psca_received(_ptr(S), _ptr(A), _ptr(g), _ptr(H), _ptr(Z), B, L, N, K, M,
                             _ptr(Y), _stream(torch)), "psca_received")
    return Y


def empirical_cov_t(Y, n_antennas: int):
    """Sigma_hat = Y Y^H / M for a device tensor Y (B,L,M); returns (B,L,L)."""
    torch = _torch()
    lib = load()
    Y = Y.to(torch.complex128).contiguous()
    B, L, Mc = Y.shape
    out = torch.empty((B, L, L), dtype=torch.complex128, device=Y.device)
    _check(lib.psca_empirical_cov(_ptr(Y), B, L, Mc, int(n_antennas), _ptr(out), _stream(torch)),
           "psca_empirical_cov")
    return out


def cov_unknown_t(S, W, Nz):
    """Sigma = S diag(W) S^H + sigma^2 I for device tensors S (B,L,N) c128, W (B,N), Nz (B,)."""
    torch = _torch()
    lib = load()
    B, L, N = S.shape
    out = torch.empty((B, L, L), dtype=torch.complex128, device=S.device)
    ws = _workspace(torch, lib.psca_cov_workspace_bytes(B, N, L), S.device)
    _check(lib.psca_cov_unknown(_ptr(S), _ptr(W), _ptr(Nz), B, N, L, _ptr(out), _ptr(ws),
                                ctypes.c_size_t(ws.numel()), _stream(torch)), "psca_cov_unknown")
    return out


def hpd_inverse_t(X):
    """(inverse, status, cond_est, logdet) device tensors for Hermitian PD X (B,L,L)."""
    torch = _torch()
    lib = load()
    B, L, _ = X.shape
    out = torch.empty_like(X)
    status = torch.empty(B, dtype=torch.int32, device=X.device)
    cond = torch.empty(B, dtype=torch.float64, device=X.device)
    logdet = torch.empty(B, dtype=torch.float64, device=X.device)
    ws = _workspace(torch, lib.psca_inverse_workspace_bytes(B, L), X.device)
    _check(lib.psca_hpd_inverse(_ptr(X), B, L, _ptr(out), _ptr(status), _ptr(cond), _ptr(logdet),
                                _ptr(ws), ctypes.c_size_t(ws.numel()), _stream(torch)),
           "psca_hpd_inverse")
    return out, status, cond, logdet


def quad_forms_t(S, P, E):
    """(q, r) device tensors (B,N) for S (B,L,N), P = Sigma^-1 and E = Sigma_hat (B,L,L)."""
    torch = _torch()
    lib = load()
    B, L, N = S.shape
    q = torch.empty((B, N), dtype=torch.float64, device=S.device)
    r = torch.empty((B, N), dtype=torch.float64, device=S.device)
    ws = _workspace(torch, lib.psca_quad_workspace_bytes(B, N, L), S.device)
    _check(lib.psca_quad_forms(_ptr(S), _ptr(P), _ptr(E), B, N, L, _ptr(q), _ptr(r), _ptr(ws),
                               ctypes.c_size_t(ws.numel()), _stream(torch)), "psca_quad_forms")
    return q, r


def eval_objective_t(X, P, E):
    """(value, status) device tensors (B,) of log|Sigma| + tr(Sigma^-1 Sigma_hat)."""
    torch = _torch()
    lib = load()
    B, L, _ = X.shape
    out = torch.empty(B, dtype=torch.float64, device=X.device)
    status = torch.empty(B, dtype=torch.int32, device=X.device)
    ws = _workspace(torch, lib.psca_objective_workspace_bytes(B, L), X.device)
    _check(lib.psca_eval_objective(_ptr(X), _ptr(P), _ptr(E), B, L, _ptr(out), _ptr(status),
                                   _ptr(ws), ctypes.c_size_t(ws.numel()), _stream(torch)),
           "psca_eval_objective")
    return out, status


def prior_terms_t(kind: str, X, n_antennas: int, *, prior_lin=None, prior_p=None,
                  eff_prior=None, prior_c1=None, prior_c2=None, want_value=False,
                  want_density=False):
    """Prior gradient (B,N) [, value (B,)] [, density (B,N)] at device iterates X (B,N)."""
    torch = _torch()
    lib = load()
    dev = X.device
    B, N = X.shape
    X = X.to(torch.float64).contiguous()
    keep = []

    def t(a, dt=torch.float64):
        if a is None:
            return 0
        v = _dev(torch, a, dt, dev)
        keep.append(v)
        return v.data_ptr()

    grad = torch.empty((B, N), dtype=torch.float64, device=dev)
    val = torch.empty(B, dtype=torch.float64, device=dev) if want_value else None
    dens = torch.empty((B, N), dtype=torch.float64, device=dev) if want_density else None
    c2 = prior_c2 if prior_c2 is not None else (None, None, None)
    if prior_c2 is not None and len(c2[1]) == 0:   # keep valid pointers, empty interaction
        c2 = (c2[0], np.zeros(1, np.int32), np.zeros(1))
    args = PriorArgsC(kind=KIND_CODES[kind], B=B, N=N, n_antennas=int(n_antennas),
                      x=X.data_ptr(), prior_lin=t(prior_lin), prior_p=t(prior_p),
                      eff=eff_prior_struct(eff_prior), prior_c1=t(prior_c1),
                      prior_c2_indptr=t(c2[0], torch.int32), prior_c2_indices=t(c2[1], torch.int32),
                      prior_c2_data=t(c2[2]), grad=grad.data_ptr(),
                      value=val.data_ptr() if val is not None else 0,
                      density=dens.data_ptr() if dens is not None else 0)
    _check(lib.psca_prior_terms(ctypes.byref(args), _stream(torch)), "psca_prior_terms")
    return grad, val, dens


def coord_step_t(kind: str, X, Q, R, rho: float, hi: float, *, gains=None, prior_grad=None,
                 sigma=None):
    """One coordinate step on device tensors (B,N): returns a dict with grad, coef, cand,
    x_new (B,N), update_norm (B,) and status (B,) (PSCA_QFLOOR when sigma is given and
    the q-floor guard trips)."""
    torch = _torch()
    lib = load()
    dev = X.device
    B, N = X.shape
    L = int(sigma.shape[-1]) if sigma is not None else 1
    ins = [v.to(torch.float64).contiguous() if v is not None else None
           for v in (X, Q, R, gains, prior_grad)]
    sg = sigma.to(torch.complex128).contiguous() if sigma is not None else None
    out = {k: torch.empty((B, N), dtype=torch.float64, device=dev)
           for k in ("grad", "coef", "cand", "x_new")}
    out["update_norm"] = torch.empty(B, dtype=torch.float64, device=dev)
    out["status"] = torch.empty(B, dtype=torch.int32, device=dev)
    args = CoordArgsC(kind=KIND_CODES[kind], B=B, N=N, L=L, rho=float(rho), hi=float(hi),
                      x=ins[0].data_ptr(), q=ins[1].data_ptr(), r=ins[2].data_ptr(),
                      gains=ins[3].data_ptr() if ins[3] is not None else 0,
                      prior_grad=ins[4].data_ptr() if ins[4] is not None else 0,
                      sigma=sg.data_ptr() if sg is not None else 0,
                      **{k: out[k].data_ptr() for k in ("grad", "coef", "cand", "x_new",
                                                        "update_norm", "status")})
    _check(lib.psca_coord_step(ctypes.byref(args), _stream(torch)), "psca_coord_step")
    return out


_SM_COUNT = {}


def sm_count() -> int:
    """Multiprocessors of the current CUDA device."""
    torch = _torch()
    d = torch.cuda.current_device()
    if d not in _SM_COUNT:
        _SM_COUNT[d] = torch.cuda.get_device_properties(d).multi_processor_count
    return _SM_COUNT[d]


def _cdev(torch):
    return torch.device("cuda", torch.cuda.current_device())


def cov_unknown(pilots, weights, noise):
    torch = _torch()
    pa, single = _batched(pilots, 2)
    wa = np.asarray(weights, dtype=float).reshape(pa.shape[0], pa.shape[2])
    na = np.broadcast_to(np.asarray(noise, dtype=float), (pa.shape[0],)).copy()
    dev = _cdev(torch)
    res = cov_unknown_t(_dev(torch, pa, torch.complex128, dev), _dev(torch, wa, torch.float64, dev),
                        _dev(torch, na, torch.float64, dev)).cpu().numpy()
    return res[0] if single else res


def hpd_inverse(sigma):
    """Returns (inverse, status, cond_est, logdet) as numpy arrays."""
    torch = _torch()
    sa, single = _batched(sigma, 2)
    res = tuple(t.cpu().numpy()
                for t in hpd_inverse_t(_dev(torch, sa, torch.complex128, _cdev(torch))))
    return tuple(r[0] for r in res) if single else res


def quad_forms(pilots, sigma_inv, emp_cov):
    torch = _torch()
    pa, single = _batched(pilots, 2)
    B, L, N = pa.shape
    dev = _cdev(torch)
    q, r = quad_forms_t(_dev(torch, pa, torch.complex128, dev),
                        _dev(torch, np.asarray(sigma_inv).reshape(B, L, L), torch.complex128, dev),
                        _dev(torch, np.asarray(emp_cov).reshape(B, L, L), torch.complex128, dev))
    qn, rn = q.cpu().numpy(), r.cpu().numpy()
    return (qn[0], rn[0]) if single else (qn, rn)


def eval_objective(sigma, sigma_inv, emp_cov):
    """Returns (value, status) numpy arrays."""
    torch = _torch()
    sa, single = _batched(sigma, 2)
    B, L, _ = sa.shape
    dev = _cdev(torch)
    v, s = eval_objective_t(_dev(torch, sa, torch.complex128, dev),
                            _dev(torch, np.asarray(sigma_inv).reshape(B, L, L), torch.complex128,
                                 dev),
                            _dev(torch, np.asarray(emp_cov).reshape(B, L, L), torch.complex128,
                                 dev))
    v, s = v.cpu().numpy(), s.cpu().numpy()
    return (v[0], s[0]) if single else (v, s)


def profile_begin():
    """Start per-kernel CUDA-event timing of subsequent solves on this thread."""
    _check(load().psca_profile_begin(), "psca_profile_begin")


def profile_end() -> dict:
    """Stop timing; returns summed device ms and launch counts per kernel family."""
    cms, fms = ctypes.c_double(), ctypes.c_double()
    cn, fn = ctypes.c_int(), ctypes.c_int()
    _check(load().psca_profile_end(ctypes.byref(cms), ctypes.byref(cn), ctypes.byref(fms),
                                   ctypes.byref(fn)), "psca_profile_end")
    return {"column_ms": cms.value, "column_launches": cn.value, "factor_ms": fms.value,
            "factor_launches": fn.value}


def set_serial(on: bool) -> None:
    """Issue every launch of later solves on the caller's stream (serialised profiling)."""
    _check(load().psca_set_serial(int(bool(on))), "psca_set_serial")


def profile_launches() -> list:
    """[(kind, ms)] of every launch recorded since profile_begin (0 column, 1 factor)."""
    lib = load()
    n = lib.psca_profile_launches(None, None, 0)
    if n < 0:
        _check(n, "psca_profile_launches")
    ms = (ctypes.c_double * max(n, 1))()
    kinds = (ctypes.c_int * max(n, 1))()
    rc = lib.psca_profile_launches(ms, kinds, n)
    if rc < 0:
        _check(rc, "psca_profile_launches")
    return [(kinds[i], ms[i]) for i in range(n)]


def version() -> str:
    return load().psca_version().decode()


def finite_or_inf(v: float) -> float:
    return v if math.isfinite(v) else math.inf
