"""TEST-ONLY numpy restatement of the three DDRGF phases of csrc/ddrgf.cu, with the
same packet layout, so the distributed protocol (paper_2605_19910_b200/distributed.py)
can run under torch.distributed/gloo on a CPU-only host. Not importable by the product."""
import numpy as np
import torch

from paper_2605_19910_b200.distributed import PACKET_BLOCKS, PHASE2_BLOCKS, layer_range, partition

GAMMA = 1.0


def _blk(T, i, off):  # slot memory -> (row, col)
    return T[i, off + 1].numpy().T


def _put(T, i, off, m):
    T[i, off + 1] = torch.from_numpy(np.ascontiguousarray(m.T))


def _slot(m):
    return np.ascontiguousarray(m.T)


def _rgf_chain(diag, up, lo):
    n = len(diag)
    X = [None] * n
    X[n - 1] = np.linalg.inv(diag[n - 1])
    for i in range(n - 2, -1, -1):
        X[i] = np.linalg.inv(diag[i] - up[i] @ X[i + 1] @ lo[i])
    G, Gu, Gl = [None] * n, [None] * (n - 1), [None] * (n - 1)
    G[0] = X[0]
    for i in range(1, n):
        um, lm = up[i - 1] @ X[i], X[i] @ lo[i - 1]
        Gu[i - 1] = -G[i - 1] @ um
        Gl[i - 1] = -lm @ G[i - 1]
        G[i] = X[i] - lm @ Gu[i - 1]
    return G, Gu, Gl


class NumpyPhases:
    def __init__(self, l, b, s2):
        self.l, self.b, self.s2 = l, b, s2
        self.tasks = partition(l, s2)

    def phase1(self, A_loc, t0, t1):
        b = self.b
        L0, _ = layer_range(self.tasks, t0, t1)
        A = lambda a, off: _blk(A_loc, a - L0, off)  # noqa: E731
        pk = np.zeros((t1 - t0, PACKET_BLOCKS, b, b), dtype=np.complex128)
        for t in range(t0, t1):
            tk = self.tasks[t]
            q = t - t0
            if tk.count:
                n = tk.count
                M = np.zeros((n * b, n * b), dtype=complex)
                for i in range(n):
                    M[i * b:(i + 1) * b, i * b:(i + 1) * b] = A(tk.first + i, 0)
                    if i + 1 < n:
                        M[i * b:(i + 1) * b, (i + 1) * b:(i + 2) * b] = A(tk.first + i, 1)
                        M[(i + 1) * b:(i + 2) * b, i * b:(i + 1) * b] = A(tk.first + i + 1, -1)
                g = GAMMA * (np.abs(A(tk.sep, 0)).max() or 1.0)
                M[:b, :b] += 1j * g * np.eye(b)
                M[-b:, -b:] += 1j * g * np.eye(b)
                Mi = np.linalg.inv(M)
                corners = (Mi[:b, :b], Mi[:b, -b:], Mi[-b:, :b], Mi[-b:, -b:])
                for k, m in enumerate(corners):
                    pk[q, k] = _slot(m)
                pk[q, 6] = _slot(A(tk.sep - 1, 1))
            x0 = tk.first if tk.count else tk.sep
            pk[q, 4] = _slot(A(tk.sep, 0))
            pk[q, 5] = _slot(A(tk.sep, -1))
            pk[q, 7] = _slot(A(tk.sep, 1))
            pk[q, 8] = _slot(A(x0, -1))
        return torch.from_numpy(pk)

    def phase2(self, packets):
        b, T = self.b, len(self.tasks)
        P = lambda t, k: packets[t, k].numpy().T  # noqa: E731
        I = np.eye(b)
        gam = [GAMMA * (np.abs(P(t, 4)).max() or 1.0) for t in range(T)]  # per-task fake-lead strength
        out = np.zeros((T, PHASE2_BLOCKS, b, b), dtype=np.complex128)
        gL, Y = [None] * T, [None] * T
        for t, tk in enumerate(self.tasks):
            g = gam[t]
            if tk.count:
                SL = P(t, 8) @ gL[t - 1] @ P(t - 1, 7) if t > 0 else np.zeros((b, b), complex)
                out[t, 0] = _slot(SL)
                Df = SL + 1j * g * I
                e1 = P(t, 3) + P(t, 2) @ np.linalg.inv(I - Df @ P(t, 0)) @ Df @ P(t, 1)
                gld = e1 + 1j * g * e1 @ np.linalg.inv(I - 1j * g * e1) @ e1
                Sleft = P(t, 5) @ gld @ P(t, 6)
            else:
                Sleft = P(t, 5) @ gL[t - 1] @ P(t - 1, 7)
                out[t, 0] = _slot(Sleft)
            gL[t] = np.linalg.inv(P(t, 4) - Sleft)
            out[t, 3] = _slot(gL[t])
        for t in range(T - 1, -1, -1):
            tk = self.tasks[t]
            g = gam[t]
            SR = P(t, 7) @ Y[t + 1] @ P(t + 1, 8) if t < T - 1 else np.zeros((b, b), complex)
            out[t, 1] = _slot(SR)
            gR = np.linalg.inv(P(t, 4) - SR)
            if tk.count:
                Dl = P(t, 6) @ gR @ P(t, 5) + 1j * g * I
                a1 = P(t, 0) + P(t, 1) @ np.linalg.inv(I - Dl @ P(t, 3)) @ Dl @ P(t, 2)
                Y[t] = a1 + 1j * g * a1 @ np.linalg.inv(I - 1j * g * a1) @ a1
            else:
                Y[t] = gR
            out[t, 2] = _slot(Y[t])
        return torch.from_numpy(out)

    def phase3(self, A_loc, out, t0, t1):
        T = len(self.tasks)
        L0, _ = layer_range(self.tasks, t0, t1)
        A = lambda a, off: _blk(A_loc, a - L0, off)  # noqa: E731
        O_ = lambda t, k: out[t, k].numpy().T  # noqa: E731
        G = torch.zeros_like(A_loc)
        for t in range(t0, t1):
            tk = self.tasks[t]
            layers = list(range(tk.first, tk.first + tk.count)) + [tk.sep]
            diag = [A(x, 0).copy() for x in layers]
            if t > 0:
                diag[0] = diag[0] - O_(t, 0)
            if t < T - 1:
                diag[-1] = diag[-1] - O_(t, 1)
            up = [A(x, 1) for x in layers[:-1]]
            lo = [A(x + 1, -1) for x in layers[:-1]]
            g, gu, gl = _rgf_chain(diag, up, lo)
            for q, x in enumerate(layers):
                _put(G, x - L0, 0, g[q])
                if q + 1 < len(layers):
                    _put(G, x - L0, 1, gu[q])
                    _put(G, x + 1 - L0, -1, gl[q])
        return G

    def halo(self, G, t0, t1):
        L0, _ = layer_range(self.tasks, t0, t1)
        tk0, tk1 = self.tasks[t0], self.tasks[t1 - 1]
        x0 = tk0.first if tk0.count else tk0.sep
        return torch.stack([G[x0 - L0, 1].clone(), G[tk1.sep - L0, 1].clone()])

    def couplings(self, A_loc, G, out, t0, t1, prev_sep_g=None, next_x0_g=None):
        T = len(self.tasks)
        L0, _ = layer_range(self.tasks, t0, t1)
        A = lambda a, off: _blk(A_loc, a - L0, off)  # noqa: E731
        O_ = lambda t, k: out[t, k].numpy().T  # noqa: E731
        x0_of = lambda t: self.tasks[t].first if self.tasks[t].count else self.tasks[t].sep  # noqa: E731
        for t in range(t0, t1):
            x0 = x0_of(t)
            if t > 0:
                gss = prev_sep_g.numpy().T if t == t0 else _blk(G, self.tasks[t - 1].sep - L0, 0)
                _put(G, x0 - L0, -1, -O_(t, 2) @ A(x0, -1) @ gss)
            if t < T - 1:
                sp = self.tasks[t].sep
                gxx = next_x0_g.numpy().T if t == t1 - 1 else _blk(G, x0_of(t + 1) - L0, 0)
                _put(G, sp - L0, 1, -O_(t, 3) @ A(sp, 1) @ gxx)
        return G
