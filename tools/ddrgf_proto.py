"""Numpy prototype of the stabilised DDRGF used by the GPU path (design check only).

Domains / separators follow interleave_permutation(layout, 1, s2) (partition.hpp:39-75).
Phase 1: corners (a, b, c, e) of each domain inverse with FAKE absorbing leads
         -i*gamma*I on its first and last block (well conditioned).
Phase 2: left-/right-connected sweeps over the separators; the true boundary
         self-energies enter through a 2b x 2b Woodbury correction of the corners.
Phase 3: plain RGF re-solve of every domain + its right separator with the exact
         boundary self-energies; separator couplings from the right-connected G.
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from oracle import bbsi_oracle as O  # noqa: E402


def inv(x):
    return np.linalg.inv(x)


def rgf_chain(diag, up, lo):
    """Selected inverse of a block tridiagonal chain given as lists: diag[i], up[i]=A[i,i+1], lo[i]=A[i+1,i]."""
    n = len(diag)
    if n == 1:
        return [inv(diag[0])], [], []
    X = [None] * n
    S = diag[n - 1]
    X[n - 1] = inv(S)
    for i in range(n - 2, -1, -1):
        S = diag[i] - up[i] @ X[i + 1] @ lo[i]
        X[i] = inv(S)
    # downward (reference form with umult/lmult)
    G = [None] * n
    Gu = [None] * (n - 1)
    Gl = [None] * (n - 1)
    G[0] = X[0]
    for i in range(1, n):
        um = up[i - 1] @ X[i]
        lm = X[i] @ lo[i - 1]
        Gu[i - 1] = -G[i - 1] @ um
        Gl[i - 1] = -lm @ G[i - 1]
        G[i] = X[i] - lm @ Gu[i - 1]
    return G, Gu, Gl


def corners(diag, up, lo, sig0):
    """(a, b, c, e) of inv(A_d - E_f sig0 E_f' - E_l sig0 E_l')."""
    d = [x.copy() for x in diag]
    d[0] = d[0] - sig0
    d[-1] = d[-1] - sig0
    n = len(d)
    # dense for the prototype (GPU: RGF + first-row/col recurrences)
    b = d[0].shape[0]
    M = np.zeros((n * b, n * b), dtype=complex)
    for i in range(n):
        M[i * b:(i + 1) * b, i * b:(i + 1) * b] = d[i]
        if i + 1 < n:
            M[i * b:(i + 1) * b, (i + 1) * b:(i + 2) * b] = up[i]
            M[(i + 1) * b:(i + 2) * b, i * b:(i + 1) * b] = lo[i]
    Mi = inv(M)
    return (Mi[:b, :b], Mi[:b, -b:], Mi[-b:, :b], Mi[-b:, -b:])


def woodbury_ll(K, sig0, sigL):
    """[inv(Atilde + E_f(sig0 - sigL)E_f' + E_l sig0 E_l')]_{l,l} from corners K."""
    a, b_, c, e = K
    bsz = a.shape[0]
    Kf = np.block([[a, b_], [c, e]])
    D = np.zeros((2 * bsz, 2 * bsz), dtype=complex)
    D[:bsz, :bsz] = sigL - sig0
    D[bsz:, bsz:] = -sig0
    W = inv(np.eye(2 * bsz) - D @ Kf) @ D
    return e + np.hstack([c, e]) @ W @ np.vstack([b_, e])


def woodbury_ff(K, sig0, sigR):
    a, b_, c, e = K
    bsz = a.shape[0]
    Kf = np.block([[a, b_], [c, e]])
    D = np.zeros((2 * bsz, 2 * bsz), dtype=complex)
    D[:bsz, :bsz] = -sig0
    D[bsz:, bsz:] = sigR - sig0
    W = inv(np.eye(2 * bsz) - D @ Kf) @ D
    return a + np.hstack([a, b_]) @ W @ np.vstack([a, c])


def ddrgf_stable(m: O.Band, s2: int, gamma: float = 1.0):
    lay = m.layout
    l, b = lay.num_layers, lay.block_sizes[0]
    order, desc = O.interleave_permutation(lay, 1, s2)
    T = desc.n_tasks()
    sig0 = -1j * gamma * np.eye(b)
    A = lambda a, off: m.block(a, off)  # noqa: E731
    dom = desc.interior_groups
    sep = [g[0] for g in desc.separator_groups]
    K = [None] * T
    for i, (f, cnt) in enumerate(dom):
        if cnt:
            K[i] = corners([A(f + q, 0) for q in range(cnt)], [A(f + q, 1) for q in range(cnt - 1)],
                           [A(f + q + 1, -1) for q in range(cnt - 1)], sig0)
    # left sweep
    gL = [None] * T
    gLdom = [None] * T
    sigL = [None] * T
    for i, (f, cnt) in enumerate(dom):
        s = sep[i]
        if cnt:
            sigL[i] = np.zeros((b, b), complex) if i == 0 else A(f, -1) @ gL[i - 1] @ A(f - 1, 1)
            gLdom[i] = woodbury_ll(K[i], sig0, sigL[i])
            gL[i] = inv(A(s, 0) - A(s, -1) @ gLdom[i] @ A(s - 1, 1))
        else:
            gL[i] = inv(A(s, 0) - A(s, -1) @ gL[i - 1] @ A(s - 1, 1)) if i > 0 else inv(A(s, 0))
    # right sweep
    gR = [None] * T
    gRdom = [None] * T
    sigR = [None] * T  # on the last layer of domain i (from separator i)
    for i in range(T - 1, -1, -1):
        s = sep[i]
        if i == T - 1:
            gR[i] = inv(A(s, 0))
        else:
            fn, cn = dom[i + 1]
            if cn:
                gR[i] = inv(A(s, 0) - A(s, 1) @ gRdom[i + 1] @ A(s + 1, -1))
            else:
                gR[i] = inv(A(s, 0) - A(s, 1) @ gR[i + 1] @ A(s + 1, -1))
        f, cnt = dom[i]
        if cnt:
            lst = f + cnt - 1
            sigR[i] = A(lst, 1) @ gR[i] @ A(s, -1)
            gRdom[i] = woodbury_ff(K[i], sig0, sigR[i])
    # phase 3: re-solve domain + right separator
    g = O.Band(lay)
    Gss = [None] * T
    for i, (f, cnt) in enumerate(dom):
        s = sep[i]
        layers = list(range(f, f + cnt)) + [s]
        diag = [A(x, 0).copy() for x in layers]
        if i > 0:
            left = A(layers[0], -1) @ gL[i - 1] @ A(layers[0] - 1, 1)
            diag[0] = diag[0] - left
        if i < T - 1:
            fn, cn = dom[i + 1]
            right = A(s, 1) @ (gRdom[i + 1] if cn else gR[i + 1]) @ A(s + 1, -1)
            diag[-1] = diag[-1] - right
        up = [A(x, 1) for x in layers[:-1]]
        lo = [A(x + 1, -1) for x in layers[:-1]]
        G, Gu, Gl = rgf_chain(diag, up, lo)
        for q, x in enumerate(layers):
            g.set_block(x, 0, G[q])
            if q + 1 < len(layers):
                g.set_block(x, 1, Gu[q])
                g.set_block(x + 1, -1, Gl[q])
        Gss[i] = G[-1]
    # couplings separator i-1 <-> first layer of X_i
    for i in range(1, T):
        f, cnt = dom[i]
        x0 = f if cnt else sep[i]
        s = sep[i - 1]
        gr = gRdom[i] if cnt else gR[i]
        g.set_block(x0, -1, -gr @ A(x0, -1) @ Gss[i - 1])
        g.set_block(s, 1, -Gss[i - 1] @ A(s, 1) @ gr)
    return g


if __name__ == "__main__":
    from oracle import dyson_oracle as DO

    for (l, b, s2, eta, gamma) in [(32, 32, 7, 1e-4, 1.0), (64, 64, 15, 1e-4, 1.0), (64, 64, 7, 1e-5, 1.0),
                                   (96, 64, 11, 1e-4, 0.5), (96, 64, 11, 1e-4, 2.0), (40, 128, 9, 1e-4, 1.0),
                                   (23, 16, 4, 1e-3, 1.0)]:
        h = DO.hamiltonian(l, 1, b, 3)
        a = DO.dyson_matrix(h, 0.1 + 1j * eta, 1)
        ref, _ = O.rgf_tridiag(a)
        g = ddrgf_stable(a, s2, gamma)
        err = O.max_block_error(g, ref)
        e_ref = O.max_block_error(O.ddrgf(a, [s2])[0], ref)
        print(f"l={l} b={b} s2={s2} eta={eta} gamma={gamma}: stable {err:.2e}   reference-ddrgf {e_ref:.2e}")
    # dominant reference test matrices
    for lyr, s2 in [(10, 4), (11, 4), (13, 4), (40, 1), (15, 2)]:
        m = O.random_spd_like(O.make_layout(lyr, 3, 1), 500 + lyr, 2.0)
        print(lyr, s2, f"{O.max_block_error(ddrgf_stable(m, s2), O.rgf_tridiag(m)[0]):.2e}")
