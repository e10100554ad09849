"""Test doubles for the sharded decoder: a NumPy stand-in for the GPU-local
block primitives (CPU tests only) and in-process thread collectives."""
import threading

import numpy as np


class NumpyBlockBackend:
    """rhs/apply/residual/update of one column block, on host arrays."""

    def __init__(self, plan, Lr, Lc, gbar_r, gbar_c, c0, c1):
        self.p, self.n = plan.p, plan.n
        self.c0, self.c1 = c0, c1
        self.Lr, self.Lc = Lr.to_scipy(), Lc.to_scipy()
        self.gr, self.gc = gbar_r, gbar_c
        self.M = np.zeros((self.p, self.n))
        self.M[np.ix_(plan.omega_r, plan.omega_c)] = 1.0
        self.rsel = {int(r): k for k, r in enumerate(plan.omega_r)}
        self.csel = {int(c): k for k, c in enumerate(plan.omega_c)}

    @staticmethod
    def _np(a):
        return a.numpy() if hasattr(a, "numpy") else a

    def rhs(self, Xt, B):
        Xt = self._np(Xt)
        Bv = self._np(B).reshape((self.p, self.c1 - self.c0), order="F")
        Bv[:] = 0.0
        for c in range(self.c0, self.c1):
            if c in self.csel:
                for r, k in self.rsel.items():
                    Bv[r, c - self.c0] = Xt[k, self.csel[c]]
        return float(np.sum(Bv * Bv))

    def apply(self, P_full, AP):
        Pf = self._np(P_full)
        Pm = Pf[: self.p * self.n].reshape((self.p, self.n), order="F") if Pf.size >= self.p * self.n else None
        Pm = Pf.reshape((self.p, -1), order="F")[:, : self.n]
        full = self.gc * (self.Lc.T @ Pm.T).T + self.gr * (self.Lr @ Pm) + self.M * Pm
        blk = full[:, self.c0:self.c1]
        APv = self._np(AP).reshape((self.p, self.c1 - self.c0), order="F")
        APv[:] = blk
        return float(np.sum(Pm[:, self.c0:self.c1] * blk))

    def residual(self, alpha, R, AP):
        r = self._np(R)
        r -= alpha * self._np(AP)
        return float(np.sum(r * r))

    def update(self, alpha, beta, X, P, R):
        x, p, r = self._np(X), self._np(P), self._np(R)
        x += alpha * p
        p[:] = r + beta * p


class ThreadCollectives:
    """Collectives among `world` threads of one process (a barrier and
    shared slots), for running several ranks in-process."""

    class Shared:
        def __init__(self, world):
            self.world = world
            self.barrier = threading.Barrier(world)
            self.slots = [None] * world

    def __init__(self, shared, rank):
        self.s = shared
        self.rank = rank
        self.world = shared.world

    def all_gather_blocks(self, full, block):
        self.s.slots[self.rank] = block
        self.s.barrier.wait()
        chunks = full.chunk(self.world) if hasattr(full, "chunk") else np.split(full, self.world)
        for g in range(self.world):
            chunks[g][:] = self.s.slots[g]
        self.s.barrier.wait()

    def allreduce_sum(self, value, like=None):
        self.s.slots[self.rank] = float(value)
        self.s.barrier.wait()
        tot = 0.0
        for g in range(self.world):
            tot += self.s.slots[g]
        self.s.barrier.wait()
        return tot
