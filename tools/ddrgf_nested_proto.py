"""Numpy prototype of the two-level stabilised DDRGF (design check for csrc/ddrgf.cu).

Level 0: tasks t = [domain D_t, separator s_t] (interleave_permutation(l, 1, s2_0)),
fake-lead corners K_t = (a, b, c, e) of every domain (fake absorbing leads +i*g_t on its
first and last block). Level 1 (the reference's ddrgf_level recursion on the separator
chain, ddrgf.hpp:363-369): groups of s2_1 level-0 separators + 1 level-1 separator, i.e.
super-domains [D_ta, s_ta, ..., s_{tb-1}, D_tb] with the level-1 separator s_tb.

  merge:     the fake-lead corners of every super-domain from its members' corners
             (2-port concatenation through a separator: a 3b x 3b Woodbury system in the
             interface blocks {l1, s, f2}; no isolated-domain inverse is formed);
  phase 2^1: left/right sweeps over the level-1 separators (the single-level phase 2 on
             the super-domains' packets) -> Sigma at every super-domain boundary;
  phase 2^0: inside every super-domain (independent of each other), the level-0 sweeps
             with the level-1 boundary values -> Sigma at every level-0 interface;
  phase 3:   unchanged (chains re-solved with exact boundary self-energies).
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from oracle import bbsi_oracle as O  # noqa: E402
from oracle import dyson_oracle as DO  # noqa: E402
from paper_2605_19910_b200.distributed import partition  # noqa: E402

inv = np.linalg.inv


def corners(m, first, count, g):
    b = m.block(first, 0).shape[0]
    M = np.zeros((count * b, count * b), dtype=complex)
    for i in range(count):
        M[i * b:(i + 1) * b, i * b:(i + 1) * b] = m.block(first + i, 0)
        if i + 1 < count:
            M[i * b:(i + 1) * b, (i + 1) * b:(i + 2) * b] = m.block(first + i, 1)
            M[(i + 1) * b:(i + 2) * b, i * b:(i + 1) * b] = m.block(first + i + 1, -1)
    M[:b, :b] += 1j * g * np.eye(b)
    M[-b:, -b:] += 1j * g * np.eye(b)
    Mi = inv(M)
    return [Mi[:b, :b], Mi[:b, -b:], Mi[-b:, :b], Mi[-b:, -b:]]


def merge(KX, gXl, A_l1s, A_sl1, A_ss, gs, A_sf2, A_f2s, KY, gYf):
    """Corners of [X, s, Y] with the fake leads of X's right end, s and Y's left end removed."""
    a1, b1, c1, e1 = KX
    a2, b2, c2, e2 = KY
    b = a1.shape[0]
    I = np.eye(b)
    Z = np.zeros((b, b), complex)
    g_s = inv(A_ss + 1j * gs * I)
    U = np.block([[-1j * gXl * I, A_l1s, Z], [A_sl1, -1j * gs * I, A_sf2], [Z, A_f2s, -1j * gYf * I]])
    D = np.block([[e1, Z, Z], [Z, g_s, Z], [Z, Z, a2]])
    W = inv(np.eye(3 * b) + U @ D) @ U
    W11, W13, W31, W33 = W[:b, :b], W[:b, 2 * b:], W[2 * b:, :b], W[2 * b:, 2 * b:]
    return [a1 - b1 @ W11 @ c1, -b1 @ W13 @ b2, -c2 @ W31 @ c1, e2 - c2 @ W33 @ b2]


def rgf_chain(diag, up, lo):
    n = len(diag)
    X = [None] * n
    X[n - 1] = inv(diag[n - 1])
    for i in range(n - 2, -1, -1):
        X[i] = inv(diag[i] - up[i] @ X[i + 1] @ lo[i])
    G, Gu, Gl = [None] * n, [None] * (n - 1), [None] * (n - 1)
    G[0] = X[0]
    for i in range(1, n):
        um, lm = up[i - 1] @ X[i], X[i] @ lo[i - 1]
        Gu[i - 1] = -G[i - 1] @ um
        Gl[i - 1] = -lm @ G[i - 1]
        G[i] = X[i] - lm @ Gu[i - 1]
    return G, Gu, Gl


def sweeps(pk, gl, gr, left_gL=None, left_An=None, right_SR=None):
    """Phase-2 sweeps over a chain of 2-ports. pk[t] = dict(K=(a,b,c,e) or None, ASS, ASL,
    ALS, ASN, AX0); gl/gr: fake-lead strengths at each 2-port's first / last block.
    Boundary: left_gL / left_An (gL of the separator before task 0 and its coupling to
    task 0's first layer), right_SR (Sigma^R on the last separator). Returns per task
    (SL, SR, Y, gL)."""
    T = len(pk)
    b = pk[0]["ASS"].shape[0]
    I = np.eye(b)
    out = [dict() for _ in range(T)]
    gL_prev, An_prev = left_gL, left_An
    for t in range(T):
        p = pk[t]
        if p["K"] is not None:
            a, b_, c, e = p["K"]
            SL = p["AX0"] @ gL_prev @ An_prev if gL_prev is not None else np.zeros((b, b), complex)
            out[t]["SL"] = SL
            Df = SL + 1j * gl[t] * I
            e1 = e + c @ inv(I - Df @ a) @ Df @ b_
            gld = e1 + 1j * gr[t] * e1 @ inv(I - 1j * gr[t] * e1) @ e1
            Sleft = p["ASL"] @ gld @ p["ALS"]
        else:
            Sleft = p["ASL"] @ gL_prev @ An_prev
            out[t]["SL"] = Sleft
        out[t]["gL"] = inv(p["ASS"] - Sleft)
        gL_prev, An_prev = out[t]["gL"], p["ASN"]
    Ynext = None
    for t in range(T - 1, -1, -1):
        p = pk[t]
        if t < T - 1:
            SR = p["ASN"] @ Ynext @ pk[t + 1]["AX0"]
        else:
            SR = right_SR if right_SR is not None else np.zeros((b, b), complex)
        out[t]["SR"] = SR
        gR = inv(p["ASS"] - SR)
        if p["K"] is not None:
            a, b_, c, e = p["K"]
            Dl = p["ALS"] @ gR @ p["ASL"] + 1j * gr[t] * I
            a1 = a + b_ @ inv(I - Dl @ e) @ Dl @ c
            Y = a1 + 1j * gl[t] * a1 @ inv(I - 1j * gl[t] * a1) @ a1
        else:
            Y = gR
        out[t]["Y"] = Y
        Ynext = Y
    return out


def ddrgf_two_level(m, s2_0, s2_1, gamma0=1.0):
    l = m.num_layers
    A = m.block
    tasks = partition(l, s2_0)
    T = len(tasks)
    gam = [gamma0 * (np.abs(A(tk.sep, 0)).max() or 1.0) for tk in tasks]
    pk = []
    for t, tk in enumerate(tasks):
        x0 = tk.first if tk.count else tk.sep
        pk.append(dict(K=corners(m, tk.first, tk.count, gam[t]) if tk.count else None, ASS=A(tk.sep, 0),
                       ASL=A(tk.sep, -1) if tk.sep > 0 else None, ALS=A(tk.sep - 1, 1) if tk.count else None,
                       ASN=A(tk.sep, 1) if tk.sep + 1 < l else None, AX0=A(x0, -1) if x0 > 0 else None))
    # level-1 groups over the T separators (partition of a chain of T layers)
    groups = partition(T, s2_1)
    sup, gl1, gr1 = [], [], []
    for grp in groups:
        ta, tb = grp.first, grp.sep  # member tasks ta..tb, level-1 separator = s_tb
        K = pk[ta]["K"]
        for t in range(ta, tb):  # merge through separator s_t with task t+1
            K = merge(K, gam[t], pk[t]["ALS"], pk[t]["ASL"], pk[t]["ASS"], gam[t], pk[t]["ASN"], pk[t + 1]["AX0"],
                      pk[t + 1]["K"], gam[t + 1])
        sup.append(dict(K=K, ASS=pk[tb]["ASS"], ASL=pk[tb]["ASL"], ALS=pk[tb]["ALS"], ASN=pk[tb]["ASN"],
                        AX0=pk[ta]["AX0"]))
        gl1.append(gam[ta])
        gr1.append(gam[tb])
    out1 = sweeps(sup, gl1, gr1)
    out0 = [None] * T
    for u, grp in enumerate(groups):
        ta, tb = grp.first, grp.sep
        left_gL = out1[u - 1]["gL"] if u > 0 else None
        left_An = pk[ta - 1]["ASN"] if u > 0 else None
        right_SR = out1[u]["SR"] if u < len(groups) - 1 else None
        o = sweeps(pk[ta:tb + 1], gam[ta:tb + 1], gam[ta:tb + 1], left_gL, left_An, right_SR)
        for k, t in enumerate(range(ta, tb + 1)):
            out0[t] = o[k]
    # phase 3 + couplings (as the single-level engine)
    g = O.Band(m.layout)
    for t, tk in enumerate(tasks):
        layers = list(range(tk.first, tk.first + tk.count)) + [tk.sep]
        diag = [A(x, 0).copy() for x in layers]
        if t > 0:
            diag[0] = diag[0] - out0[t]["SL"]
        if t < T - 1:
            diag[-1] = diag[-1] - out0[t]["SR"]
        Gc, Gu, Gl = rgf_chain(diag, [A(x, 1) for x in layers[:-1]], [A(x + 1, -1) for x in layers[:-1]])
        for q, x in enumerate(layers):
            g.set_block(x, 0, Gc[q])
            if q + 1 < len(layers):
                g.set_block(x, 1, Gu[q])
                g.set_block(x + 1, -1, Gl[q])
    for t, tk in enumerate(tasks):
        x0 = tk.first if tk.count else tk.sep
        if t > 0:
            s = tasks[t - 1].sep
            g.set_block(x0, -1, -out0[t]["Y"] @ A(x0, -1) @ g.block(s, 0))
        if t < T - 1:
            nx = tasks[t + 1].first if tasks[t + 1].count else tasks[t + 1].sep
            g.set_block(tk.sep, 1, -out0[t]["gL"] @ A(tk.sep, 1) @ g.block(nx, 0))
    return g


if __name__ == "__main__":
    for (l, b, s20, s21, E, eta) in [(15, 8, 4, 2, 0.2, 1e-3), (40, 16, 4, 2, 0.1, 1e-4), (63, 16, 3, 3, -0.4, 1e-4),
                                     (100, 32, 5, 2, 0.1, 1e-4), (31, 8, 1, 1, 0.3, 1e-3), (77, 16, 4, 4, 0.05, 1e-5)]:
        a = DO.dyson_matrix(DO.hamiltonian(l, 1, b, 7), complex(E, eta), 1)
        ref, _ = O.rgf_tridiag(a)
        g = ddrgf_two_level(a, s20, s21)
        print(f"l={l} b={b} plan=({s20},{s21}) E={E} eta={eta}: max block error vs RGF "
              f"{O.max_block_error(g, ref):.2e}")
    for lyr, plan in [(15, (4, 2)), (21, (4, 2)), (8, (1, 1)), (40, (2, 3))]:
        m = O.random_spd_like(O.make_layout(lyr, 3, 1), 500 + lyr, 2.0)
        print(lyr, plan, f"{O.max_block_error(ddrgf_two_level(m, *plan), O.rgf_tridiag(m)[0]):.2e}")
