"""CPU oracle (TEST INFRASTRUCTURE ONLY): Krylov solvers.

* `cg_solve` restates the reference's unpreconditioned CG
  (`warpkit/kernels.py:283-331`) statement for statement: x updated before r,
  true residual `b - A x` every 50th iteration (kernels.py:322-323), strict
  `hist[-1] > tol*||b||` loop test (kernels.py:314), `BreakdownError` when
  p.Ap <= 0 (kernels.py:317-318), zero-rhs early return (kernels.py:311-312),
  `len(hist) == iterations + 1`. With the bitwise SpMV of `sparse_ref.spmv`
  swapped in it reproduces the reference's histories bit for bit (pinned by
  `tests/golden/cg_*.npz`).
* `bicgstab_solve` and `gmres_solve` have NO reference implementation
  (SPEC.md:15, 367 list them as non-goals): they are textbook restatements
  (van der Vorst BiCGSTAB; restarted GMRES(m) with classical Gram-Schmidt,
  Givens rotations and a true-residual restart) that fix the update order
  the B200 solvers follow. Parity for them is "unpinned" by the reference.

The `spmv` argument is any callable `v -> A v`; `dot` defaults to numpy's
`@` (OpenBLAS ddot, as in the reference).
"""

import math

import numpy as np


class BreakdownError(Exception):
    """Mirror of warpkit.errors.BreakdownError (errors.py:59-60)."""


def _dot(a, b):
    return float(a @ b)


def cg_solve(spmv, b, tol, max_iters, dot=_dot, replace_every=50):
    """kernels.py:283-331 restated; returns (x, residual_history)."""
    b = np.asarray(b, dtype=np.float64)
    if tol <= 0:
        raise ValueError("tol must be positive")
    b_norm = float(np.linalg.norm(b))
    x = np.zeros_like(b)
    r = b.copy()
    p = b.copy()
    rho = dot(b, b)
    hist = [b_norm]
    if b_norm == 0.0:
        return x, np.asarray(hist)
    threshold = tol * b_norm
    it = 0
    while it < max_iters and hist[-1] > threshold:
        q = spmv(p)
        p_ap = dot(p, q)
        if p_ap <= 0.0:
            raise BreakdownError(f"p.Ap = {p_ap} at iteration {it + 1}; system is not SPD")
        alpha = rho / p_ap
        x = x + alpha * p
        it += 1
        if replace_every and it % replace_every == 0:
            r = b - spmv(x)
        else:
            r = r - alpha * q
        rho_next = dot(r, r)
        hist.append(math.sqrt(rho_next))
        beta = rho_next / rho
        p = r + beta * p
        rho = rho_next
    return x, np.asarray(hist)


def pcg_jacobi_solve(spmv, diag, b, tol, max_iters, dot=_dot, replace_every=50):
    """Jacobi-preconditioned CG: `cg_solve` (kernels.py:283-331) with
    z = r / diag (the apply_jacobi fixture, preconditioner.cu:9-17) inserted
    after every residual update; rho = r.z drives alpha and beta, the history
    and stopping test stay on ||r|| (the reference's criterion). NO reference
    PCG exists: this fixes the order the B200 solver follows."""
    b = np.asarray(b, dtype=np.float64)
    diag = np.asarray(diag, dtype=np.float64)
    if tol <= 0:
        raise ValueError("tol must be positive")
    b_norm = float(np.linalg.norm(b))
    x = np.zeros_like(b)
    r = b.copy()
    z = r / diag
    p = z.copy()
    rho = dot(r, z)
    hist = [b_norm]
    if b_norm == 0.0:
        return x, np.asarray(hist)
    threshold = tol * b_norm
    it = 0
    while it < max_iters and hist[-1] > threshold:
        q = spmv(p)
        p_ap = dot(p, q)
        if p_ap <= 0.0:
            raise BreakdownError(f"p.Ap = {p_ap} at iteration {it + 1}; system is not SPD")
        alpha = rho / p_ap
        x = x + alpha * p
        it += 1
        if replace_every and it % replace_every == 0:
            r = b - spmv(x)
        else:
            r = r - alpha * q
        z = r / diag
        rho_next = dot(r, z)
        hist.append(math.sqrt(dot(r, r)))
        beta = rho_next / rho
        p = z + beta * p
        rho = rho_next
    return x, np.asarray(hist)


def bicgstab_solve(spmv, b, tol, max_iters, dot=_dot):
    """Unpreconditioned BiCGSTAB, x0 = 0, shadow residual r^ = b.

    Per iteration (one history entry = ||r|| after the full step):
        rho_new = r^.r ;  beta = (rho_new/rho) * (alpha/omega)
        p = r + beta*(p - omega*v) ;  v = A p ;  alpha = rho_new / (r^.v)
        s = r - alpha*v ;  if ||s|| <= thr: x = x + alpha*p, hist += ||s||, stop
        t = A s ;  omega = (t.s)/(t.t)
        x = x + alpha*p + omega*s ;  r = s - omega*t ;  hist += ||r||
    Breakdown (BreakdownError) when rho_new == 0, r^.v == 0 or t.t == 0
    before convergence. Loop test mirrors CG: `hist[-1] > tol*||b||`.
    """
    b = np.asarray(b, dtype=np.float64)
    if tol <= 0:
        raise ValueError("tol must be positive")
    b_norm = math.sqrt(dot(b, b))
    x = np.zeros_like(b)
    r = b.copy()
    rhat = b.copy()
    p = np.zeros_like(b)
    v = np.zeros_like(b)
    rho = alpha = omega = 1.0
    hist = [b_norm]
    if b_norm == 0.0:
        return x, np.asarray(hist)
    thr = tol * b_norm
    it = 0
    while it < max_iters and hist[-1] > thr:
        rho_new = dot(rhat, r)
        if rho_new == 0.0:
            raise BreakdownError(f"rho = 0 at iteration {it + 1}")
        beta = (rho_new / rho) * (alpha / omega)
        p = r + beta * (p - omega * v)
        v = spmv(p)
        rv = dot(rhat, v)
        if rv == 0.0:
            raise BreakdownError(f"r^.v = 0 at iteration {it + 1}")
        alpha = rho_new / rv
        s = r - alpha * v
        it += 1
        s_norm = math.sqrt(dot(s, s))
        if s_norm <= thr:
            x = x + alpha * p
            hist.append(s_norm)
            break
        t = spmv(s)
        tt = dot(t, t)
        if tt == 0.0:
            raise BreakdownError(f"t.t = 0 at iteration {it}")
        omega = dot(t, s) / tt
        x = x + alpha * p + omega * s
        r = s - omega * t
        hist.append(math.sqrt(dot(r, r)))
        rho = rho_new
    return x, np.asarray(hist)


def givens(a, b):
    """Rotation (c, s) with [c s; -s c] [a; b] = [h; 0] (LAPACK dlartg-free
    textbook form used by the B200 solver too)."""
    if b == 0.0:
        return 1.0, 0.0
    h = math.hypot(a, b)
    return a / h, b / h


def gmres_solve(spmv, b, tol, max_iters, restart=30, dot=_dot):
    """Restarted GMRES(m), x0 = 0, classical Gram-Schmidt Arnoldi.

    Cycle: beta = ||r||, V0 = r/beta, g = beta e1. Inner step j:
        w = A V_j ; h_i = V_i.w for i <= j (batched, CGS) ;
        w = w - sum_i h_i V_i (in i order) ; h_{j+1} = ||w|| ;
        V_{j+1} = w / h_{j+1} (skipped on happy breakdown h_{j+1} == 0) ;
        apply rotations 0..j-1 to h, new rotation (c_j, s_j) = givens(h_j, h_{j+1}),
        g_{j+1} = -s_j g_j, g_j = c_j g_j ; hist += |g_{j+1}|.
    The cycle ends when |g_{j+1}| <= thr, j+1 == m, or max_iters is hit; then
    y = H^-1 g (back substitution), x = x + sum_i y_i V_i, r = b - A x, and
    the NEXT cycle's test uses the true ||r|| (which replaces the last
    history entry). Returns (x, history) with len(history) = iterations + 1.
    """
    b = np.asarray(b, dtype=np.float64)
    if tol <= 0:
        raise ValueError("tol must be positive")
    n = len(b)
    m = int(restart)
    b_norm = math.sqrt(dot(b, b))
    x = np.zeros_like(b)
    hist = [b_norm]
    if b_norm == 0.0:
        return x, np.asarray(hist)
    thr = tol * b_norm
    r = b.copy()
    beta = b_norm
    it = 0
    while it < max_iters and beta > thr:
        V = np.zeros((m + 1, n))
        H = np.zeros((m + 1, m))
        cs = np.zeros(m)
        sn = np.zeros(m)
        g = np.zeros(m + 1)
        V[0] = r / beta
        g[0] = beta
        j_done = 0
        for j in range(m):
            w = spmv(V[j])
            h = np.array([dot(V[i], w) for i in range(j + 1)])
            for i in range(j + 1):
                w = w - h[i] * V[i]
            hn = math.sqrt(dot(w, w))
            if hn != 0.0:
                V[j + 1] = w / hn
            H[: j + 1, j] = h
            H[j + 1, j] = hn
            for i in range(j):
                a, c = H[i, j], H[i + 1, j]
                H[i, j] = cs[i] * a + sn[i] * c
                H[i + 1, j] = -sn[i] * a + cs[i] * c
            cs[j], sn[j] = givens(H[j, j], H[j + 1, j])
            H[j, j] = cs[j] * H[j, j] + sn[j] * H[j + 1, j]
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            it += 1
            j_done = j + 1
            hist.append(abs(g[j + 1]))
            if abs(g[j + 1]) <= thr or it >= max_iters or hn == 0.0:
                break
        y = np.zeros(j_done)
        for i in range(j_done - 1, -1, -1):
            acc = g[i]
            for k in range(i + 1, j_done):
                acc = acc - H[i, k] * y[k]
            y[i] = acc / H[i, i]
        for i in range(j_done):
            x = x + y[i] * V[i]
        r = b - spmv(x)
        beta = math.sqrt(dot(r, r))
        hist[-1] = beta
    return x, np.asarray(hist)
