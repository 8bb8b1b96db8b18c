"""numpy model of gj_rows_kernel's block algebra (csrc/zinv.cu): blocked in-place
Gauss-Jordan inversion, two NB-column panels per step eliminated on ALL rows (thread =
physical row), one rank-2NB update M <- M(0 on P1,P2 rows / K1,K2 cols) + [W1(0 on P2)|W2]
[Vs1(0 on K2); Vs2], final scatter A^-1[i, lmap[c]] = Y[lmap[i], c]. Checks the formulas,
not the rounding:   python tools/gj_rows_proto.py"""
import numpy as np


def gj_panel(a, cand):
    """In-place GJ on the n x NB panel `a` (modified), pivots among rows with cand True.
    Returns the pivot rows in order."""
    n, nb = a.shape
    cand = cand.copy()
    src = []
    for j in range(nb):
        key = np.where(cand, np.abs(a[:, j].real) + np.abs(a[:, j].imag), -1.0)
        p = int(np.argmax(key))
        src.append(p)
        cand[p] = False
        rcp = 1.0 / a[p, j]
        u = a[p].copy()
        l = a[:, j] * rcp
        l[p] = -rcp
        x = a.copy()
        x[p] = 0
        a[:] = x - l[:, None] * u[None, :]
        a[:, j] = -l
    return src


def invert(A, nb=16):
    n = A.shape[0]
    M = A.astype(complex).copy()
    lmap = []
    used = np.zeros(n, bool)
    for k in range(0, n, 2 * nb):
        k2 = k + nb
        a = M[:, k:k2].copy()
        P1 = gj_panel(a, ~used)
        W1 = a
        used[P1] = True
        Vs1 = M[P1, :].copy()
        Vs1[:, k:k2] = np.eye(nb)
        m2 = M[:, k2:k2 + nb].copy()
        m2[P1] = 0
        m2 += W1 @ Vs1[:, k2:k2 + nb]
        P2 = gj_panel(m2, ~used)
        W2 = m2
        used[P2] = True
        raw = M[P2, :].copy()
        raw[:, k:k2] = 0
        Vs2 = raw + W1[P2] @ Vs1
        Vs2[:, k2:k2 + nb] = np.eye(nb)
        C = M.copy()
        C[P1 + P2, :] = 0
        C[:, k:k2 + nb] = 0
        W1z = W1.copy()
        W1z[P2] = 0
        Vs1z = Vs1.copy()
        Vs1z[:, k2:k2 + nb] = 0
        M = C + np.hstack([W1z, W2]) @ np.vstack([Vs1z, Vs2])
        lmap += P1 + P2
    lmap = np.array(lmap)
    out = np.empty_like(M)
    out[np.ix_(np.arange(n), lmap)] = M[lmap, :]  # A^-1[i, lmap[c]] = Y[lmap[i], c]
    return out


if __name__ == "__main__":
    rng = np.random.default_rng(0)
    for n in (64, 128, 256):
        A = rng.uniform(-1, 1, (n, n)) + 1j * rng.uniform(-1, 1, (n, n))
        X = invert(A)
        ref = np.linalg.inv(A)
        print(n, np.linalg.norm(X - ref) / np.linalg.norm(ref), np.linalg.norm(A @ X - np.eye(n)) / np.sqrt(n))
