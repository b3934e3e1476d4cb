"""Dense form of an assembled implicit operator, for the LU-SGS known-answer
tests (reference pkg/tests/test_implicit.py:160-187 solve the factored
system (D + L) D^-1 (D + U) densely and compare with lusgs_solve).

Test infrastructure: built from the operator fields the drop-in
``ImplicitOperator`` exposes (w, b, rho, u, face radii, diagonals); the
block formulas are reference implicit.py:246-326 and lusgs.py:24-59.
"""

import numpy as np


def _np(x):
    return x.detach().cpu().numpy() if hasattr(x, "detach") else np.asarray(x)


def half_block(op, cell, S, lam, sign, n):
    """A = 1/2 (w a^T + v b^T + (U + sign lam) I) of the neighbour `cell`
    across the face with area vector S (lusgs.py:24-59)."""
    w = _np(op.w)[cell][:n]
    b = _np(op.b)[cell][:n]
    rho = float(_np(op.rho)[cell])
    U = float(_np(op.u)[cell] @ S)
    a = np.zeros(n)
    a[0] = -U / rho
    a[1:4] = S / rho
    v = np.zeros(n)
    v[1:4] = S
    v[4] = U
    return 0.5 * (np.outer(w, a) + np.outer(v, b) + (U + sign * lam) * np.eye(n))


def offdiag_block(op, grid, cell, d, upper):
    """Coupling block of `cell` to its lower (upper=False) or upper neighbour
    in direction d (implicit.py:262-292)."""
    nb = list(cell)
    nb[d] += 1 if upper else -1
    f = list(cell)
    if upper:
        f[d] += 1
    nb, f = tuple(nb), tuple(f)
    S = grid.face_areas(d)[f]
    lam = float(_np(op.lam_face[d])[f])
    n = op.nvar
    sign = -1.0 if upper else 1.0
    if op.mode == "CI":
        A = half_block(op, nb, S, lam, sign, n)
        return A if upper else -A
    out = np.zeros((n, n))
    A = half_block(op, nb, S, lam, sign, 5)
    out[:5, :5] = A if upper else -A
    lam_sp = float(_np(op.lam_face_sp[d])[f])
    U = float(_np(op.u)[nb] @ S)
    c = op.sp_scale * (U + sign * lam_sp)
    out[5:, 5:] = np.eye(n - 5) * (c if upper else -c)
    return out


def diag_block(op, cell):
    """Diagonal block (implicit.py:294-302): d I, CI with chemistry minus
    V dOmega on the species rows, CS the per-species diagonal."""
    n = op.nvar
    D = np.eye(n) * float(_np(op.d_scal)[cell])
    if op.mode == "CI":
        vd = op.vdom
        if vd is not None:
            D[5:, 5:] -= _np(vd)[cell]
    else:
        D[5:, 5:] = np.diag(_np(op.d_species)[cell])
    return D


def dense_factored_matrix(op, grid):
    """(D + L) D^-1 (D + U) over a small grid (implicit.py:304-326)."""
    ni, nj, nk = grid.dims
    n = op.nvar
    N = ni * nj * nk
    at = lambda i, j, k: ((i * nj + j) * nk + k) * n
    D = np.zeros((N * n, N * n))
    L = np.zeros_like(D)
    U = np.zeros_like(D)
    for i in range(ni):
        for j in range(nj):
            for k in range(nk):
                r = at(i, j, k)
                D[r:r + n, r:r + n] = diag_block(op, (i, j, k))
                for d in range(3):
                    e = [0, 0, 0]
                    e[d] = 1
                    if (i, j, k)[d] > 0:
                        c = at(i - e[0], j - e[1], k - e[2])
                        L[r:r + n, c:c + n] = offdiag_block(op, grid, (i, j, k), d, False)
                    if (i, j, k)[d] < (ni, nj, nk)[d] - 1:
                        c = at(i + e[0], j + e[1], k + e[2])
                        U[r:r + n, c:c + n] = offdiag_block(op, grid, (i, j, k), d, True)
    return (D + L) @ np.linalg.inv(D) @ (D + U)
