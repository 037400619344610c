"""Smallest eigenvalue of C - A*(lam) by Lanczos, on the device (spectral.py of the reference).

The Krylov basis Q (k_max x n, rows padded to 16-byte multiples) lives in
HBM; each step is one pattern SpMV (the Omega coefficients assembled inside
the kernel), one streaming combination and two classical Gram-Schmidt
passes (project + subtract, each a single read of the active basis) -- the
same full reorthogonalisation, applied twice, as the reference. The
tridiagonal eigenproblem (size <= 300) is solved on the host with scipy.
"""

from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass

import numpy as np
import torch
from scipy.linalg import eigh_tridiagonal

from .device import F64, default_device


@dataclass
class EigEstimate:
    value: float
    residual: float
    verified: bool
    basis_size: int


class _DeviceOp:
    """Marks a device-native operator: op(v_dev, out_dev, dot_at) -> writes out, <out, v> at slab.
    ``assembled()`` (optional) returns a cl_pattern whose slot values are the operator's,
    assembled once, for the native Lanczos loop."""

    def __init__(self, fn, assembled=None):
        self.fn = fn
        self.assembled = assembled


def _host_callback_op(apply_s, dev):
    def fn(v, out, at):
        u = apply_s(v.cpu().numpy())
        out.copy_(torch.as_tensor(np.asarray(u, dtype=np.float64)).to(dev.dev))
        dev.lincomb(None, [out, v], [0.0, 0.0], dots=[(0, 1)], at=at, N=v.numel())
    return _DeviceOp(fn)


NATIVE = True     # one device, assembled operator: run the Lanczos loop's control flow in C++
# Small operators run the whole loop as one cooperative launch (cl_lanczos_loop_fused).
FUSED = os.environ.get("CULORADS_FUSED", "1") != "0"
FUSED_MAX_N = int(os.environ.get("CULORADS_LANCZOS_FUSED_MAX", 1 << 16))


def _lanczos_native(op, n, k_max, Q, u, r, h, dev, alphas, betas):
    """The loop below through cl_lanczos_loop (same launches; bit-identical coefficients)."""
    from . import _lib
    a = _lib.LanczosArgs()
    a.n, a.k_max, a.breakdown = n, k_max, 1e-14
    a.Q, a.ldq = Q.data_ptr(), int(Q.shape[1])
    a.u, a.r, a.h = u.data_ptr(), r.data_ptr(), h.data_ptr()
    a.S = op.assembled()
    a.slab, a.host = dev.slot(520).value, dev.host.data_ptr() + 8 * 520
    a.ws, a.stream = dev.ws.data_ptr(), dev.stream.cuda_stream
    a.alphas, a.betas = alphas.ctypes.data, betas.ctypes.data
    dbeta = dev.zeros(max(k_max, 1))
    dalpha = dev.zeros(max(k_max, 1))
    a.dbeta, a.dalpha = dbeta.data_ptr(), dalpha.data_ptr()
    k = _lib.I32(0)
    global FUSED
    fused = FUSED and n <= FUSED_MAX_N and k_max <= 4096
    if fused:
        rc = dev.lib.cl_lanczos_loop_fused(ctypes.byref(a), ctypes.byref(k))
        if _lib.coop_refused(rc, "cl_lanczos_loop_fused"):
            FUSED = fused = False
        elif _lib.barrier_timeout(rc, "cl_lanczos_loop_fused"):
            FUSED = fused = False       # Q[0] (the start vector) was only read: rerun
        else:
            dev.launches += 1
            _lib.check(rc, "cl_lanczos_loop_fused")
    if not fused:
        rc = dev.lib.cl_lanczos_loop(ctypes.byref(a), ctypes.byref(k))
        dev.launches += 9 * k.value
        _lib.check(rc, "cl_lanczos_loop")
    return k.value


def _lanczos_smallest(op, n, seed, max_basis, dev, rows=None, perm=None):
    """spectral.py:28. ``rows`` = (lo, hi, n_global): this rank's block of a
    row-sharded vector; the Gram projections are all-reduced."""
    rng = np.random.default_rng(seed)
    n_all = rows[2] if rows is not None else n
    k_max = min(n_all, max_basis)
    npad = n + (n & 1)
    Q = dev.zeros(k_max, npad)
    alphas = np.zeros(k_max)
    betas = np.zeros(max(k_max - 1, 0))
    q0 = rng.standard_normal(n_all)
    q0 /= np.linalg.norm(q0)
    if perm is not None:
        q0 = q0[perm]              # locality-ordered operator: the same start vector, relabelled
    if rows is not None:
        q0 = q0[rows[0]:rows[1]]
    Q[0, :n] = torch.as_tensor(q0).to(dev.dev)
    u = dev.zeros(npad)
    r = dev.zeros(npad)
    h = dev.zeros(k_max)
    A = 500
    k = 0
    breakdown = 1e-14
    native = NATIVE and dev.world == 1 and getattr(op, "assembled", None) is not None
    if native:
        k = _lanczos_native(op, n, k_max, Q, u, r, h, dev, alphas, betas)
    while not native and k < k_max:
        qk = Q[k, :n]
        op.fn(qk, u[:n], A)
        alphas[k] = float(dev.fetch(A + 1)[A])
        if k > 0:
            dev.lincomb(r[:n], [u[:n], qk, Q[k - 1, :n]], [1.0, -alphas[k], -betas[k - 1]])
        else:
            dev.lincomb(r[:n], [u[:n], qk], [1.0, -alphas[k]])
        for _ in range(2):      # full reorthogonalisation, twice (spectral.py:55-56)
            dev.basis_project(Q, k + 1, n, r, h)
            if dev.world > 1:
                from .shard import all_reduce_sum
                all_reduce_sum(h[:k + 1], dev.group)
            dev.basis_subtract(Q, k + 1, n, h, r)
        k += 1
        dev.lincomb(None, [r[:n]], [0.0], dots=[(0, 0)], at=A + 1)
        beta = math.sqrt(float(dev.fetch(A + 2)[A + 1]))
        scale = max(float(np.abs(alphas[:k]).max()), 1.0)
        if k == k_max or beta <= breakdown * scale:
            break
        betas[k - 1] = beta
        dev.lincomb(Q[k, :n], [r[:n]], [1.0 / beta])
    theta, y = eigh_tridiagonal(alphas[:k], betas[:k - 1], select="i", select_range=(0, 0))
    theta = float(theta[0])
    v = dev.zeros(npad)
    hy = torch.as_tensor(-y[:, 0]).to(dev.dev)
    dev.basis_subtract(Q, k, n, hy, v)            # v = Q[:k]^T y
    dev.lincomb(None, [v[:n]], [0.0], dots=[(0, 0)], at=A + 2)
    vn = math.sqrt(float(dev.fetch(A + 3)[A + 2]))
    if vn > 0:
        dev.lincomb(v[:n], [v[:n]], [1.0 / vn])
    op.fn(v[:n], u[:n], A + 3)
    dev.lincomb(None, [u[:n], v[:n]], [1.0, -theta], dots=[("out", "out")], at=A + 4)
    residual = math.sqrt(float(dev.fetch(A + 5)[A + 4]))
    del Q
    return theta, residual, k


def smallest_eigenvalue(apply_s, n, tol=1e-7, seed=0, max_basis=300, dev=None, rows=None,
                        perm=None) -> EigEstimate:
    """Smallest eigenvalue of a self-adjoint operator (spectral.py:67).

    ``apply_s`` is a host callback v -> S v (numpy), or a device operator from
    ``omega_operator``. One restart from seed+1 when the Ritz residual fails.
    """
    dev = dev or default_device()
    op = apply_s if isinstance(apply_s, _DeviceOp) else _host_callback_op(apply_s, dev)
    theta, residual, k = _lanczos_smallest(op, n, seed, max_basis, dev, rows, perm)
    if residual > tol * (1.0 + abs(theta)):
        t2, r2, k2 = _lanczos_smallest(op, n, seed + 1, max_basis, dev, rows, perm)
        if r2 < residual:
            theta, residual, k = t2, r2, k2
    return EigEstimate(value=theta, residual=residual,
                       verified=residual <= tol * (1.0 + abs(theta)), basis_size=k)


def omega_operator(ops, lam_dev, c_coeff=1.0):
    """Device SpMV v -> (c_coeff*C + A*(lam)) v over Omega, with <Sv, v> reduced."""
    dev = ops.dev

    def fn(v, out, at):
        dev.spmm(ops.adj.omega, v, 1, out=out, Z=[v], dots=[("out", ("z", 0))], at=at,
                 c_coeff=c_coeff, w1=lam_dev)

    def assembled():
        """Slot values of c_coeff*C + A*(lam) assembled once (the pre-pass fn repeats per call)."""
        from . import _lib
        from .linops import padded
        om = ops.adj.omega
        P = om.struct(c_coeff=c_coeff, w1=lam_dev)
        vals = padded(torch.empty(om.nnz, dtype=F64, device=dev.dev))
        _lib.check(dev.lib.cl_pattern_assemble(ctypes.byref(P), vals.data_ptr() if om.nnz else None, dev.sp),
                   "cl_pattern_assemble")
        dev.launches += 1
        S = om.struct(c_coeff=None)          # indices/pointers; values from `vals`
        S.cv = vals.data_ptr() if om.nnz else None
        S.c_coeff = 1.0
        assembled.keep = vals                # keep the buffer alive while the loop runs
        return S
    return _DeviceOp(fn, assembled)


def dual_infeasibility(problem, ops, lam, tol=1e-7, seed=0):
    """|min(0, sigma_min(C - A*(lam)))| / (1 + ||vec C||_1) (spectral.py:82).

    Returns (value, verified, sigma_min); lam may be host or device."""
    dev = ops.dev
    if isinstance(lam, torch.Tensor):
        neg = dev.empty(ops.problem.m)
        dev.lincomb(neg, [lam.to(dev.dev)], [-1.0])
    else:
        neg = torch.as_tensor(-np.asarray(lam, dtype=np.float64)).to(dev.dev)
    rr = getattr(ops, "row_range", None)
    rows = (rr[0], rr[1], problem.n) if rr is not None else None
    n_loc = ops.problem.n
    est = smallest_eigenvalue(omega_operator(ops, neg, 1.0), n_loc, tol=tol, seed=seed, dev=dev, rows=rows,
                              perm=getattr(ops, "perm", None))
    value = abs(min(0.0, est.value)) / (1.0 + problem.c_vec_norm1)
    return value, est.verified, est.value
