"""A CPU shard with the same phase interface as paper_1411_1702_b200.sharded.GpuShard.

TEST INFRASTRUCTURE: lets the product's multi-GPU orchestrator
(`ShardedFilter` + `TorchComm`) run as world_size-2 `gloo` processes on CPU.
The per-particle math calls the C oracle (oracle/pfsmc_oracle.c) building
blocks; the exchange buffers carry the same payload layout as the device
path. Record exchange (phase C) here ships the shard's fitness vector and
every rank recomputes the sequential CDF over all shards in rank order.
"""
from __future__ import annotations

import math

import numpy as np
import torch

from oracle_ctypes import DIMS, MODELS, Oracle, OracleError, StepConfig

from paper_1411_1702_b200.sampler import Ensemble, NumericalError

O = Oracle()


def _t(a: np.ndarray):
    return torch.from_numpy(a.view(np.uint8))


class CpuShard:
    def __init__(self, sc: StepConfig, n_glob: int, rank: int, world: int):
        self.sc = sc
        self.d, self.p = DIMS[MODELS[sc.model]]
        self.rank, self.world = rank, world
        self.n = n_glob // world
        self.n0 = rank * self.n
        self.n_glob = n_glob
        self.R = (self.d + self.p + 1) // 2 * 2
        self.W = self.R + 4
        V = 2 + self.p + self.p * (self.p + 1) // 2 + self.d
        self.V = V
        self.bufs = {0: np.zeros(2), 1: np.zeros(2 * world), 2: np.zeros(2), 3: np.zeros(2 * world),
                     4: np.zeros(n_glob), 5: np.zeros(world), 6: np.zeros(V + 1), 7: np.zeros((V + 1) * world),
                     8: np.zeros(world * self.n * self.W), 9: np.zeros(self.n * self.W),
                     10: np.zeros(2 * world, dtype=np.uint32), 11: np.zeros(2 * world * world, dtype=np.uint32)}
        self._tens = {k: _t(v) for k, v in self.bufs.items()}
        self.lse_w = 0.0
        self.mu = np.zeros(self.p)
        self.cov = np.zeros((self.p, self.p))
        self.L = None
        self.anc = np.zeros(self.n, dtype=np.int64)

    def buffer(self, which):
        return self._tens[which]

    def sync(self):
        pass

    def payload_doubles(self):
        return self.W

    def count_matrix(self):
        """world x world migration counts, derived from the keyed uniforms and ranges."""
        m = np.zeros((self.world, self.world), dtype=np.uint32)
        u_all = np.array([O.draws(self.sc.seed, self.j, ng, 3, 1, 1)[0] for ng in range(self.n_glob)])
        for ng, u in enumerate(u_all):
            r = next(r for r, (a, b) in enumerate(self.ranges) if a <= u < b)
            m[r, ng // self.n] += 1
        return m

    # ---------------------------------------------------------- ensemble
    def initialize_uniform(self, th_lo, th_hi, x_lo, x_hi):
        e = O.init_uniform(self.sc.model, self.n_glob, self.sc.seed, th_lo, th_hi, x_lo, x_hi)
        sl = slice(self.n0, self.n0 + self.n)
        self.states, self.params_u = e.states[sl].copy(), e.params_u[sl].copy()
        self.lw = np.full(self.n, -math.log(float(self.n_glob)))
        self.lse_w = 0.0
        self.mu = np.zeros(self.p)

    def set_ensemble(self, e: Ensemble):
        self.states, self.params_u = np.array(e.states, dtype=float), np.array(e.params_u, dtype=float)
        self.lw = np.array(e.logw, dtype=float)
        self.lse_w = 0.0
        self.mu = np.array(e.mean_u, dtype=float)
        self.cov = np.array(e.cov_u, dtype=float)

    def get_ensemble(self):
        return Ensemble(self.states.copy(), self.params_u.copy(), self.lw - self.lse_w, self.mu.copy(), self.cov.copy())

    def step_diagnostics(self):
        return self.anc.copy(), None, 0

    # ---------------------------------------------------------- helpers
    @staticmethod
    def _partial(x, vals, sq_last):
        nn = ~np.isnan(x)
        M = np.max(x[nn]) if nn.any() else -np.inf
        if not np.isfinite(M):
            e = np.where(np.isnan(x), np.nan, 0.0)
        else:
            e = np.where(np.isnan(x), np.nan, np.where(x == -np.inf, 0.0, np.exp(x - M)))
        out = [M]
        for k in range(vals.shape[1]):
            w = e * e if (sq_last and k == vals.shape[1] - 1) else e
            out.append(np.sum(w * vals[:, k]))
        return np.array(out)

    @staticmethod
    def _combine(parts, sq_last):
        M = np.max([p[0] for p in parts])
        tot = np.zeros(len(parts[0]) - 1)
        for p in parts:
            c = 0.0 if p[0] == -np.inf else math.exp(p[0] - M)
            w = np.full(len(tot), c)
            if sq_last:
                w[-1] = c * c
            tot += w * p[1:]
        return M, tot

    def _moment_leaf(self, lw, params, states):
        dv = params - self.mu
        cols = [np.ones(len(lw))] + [dv[:, k] for k in range(self.p)]
        cols += [dv[:, r] * dv[:, q] for r in range(self.p) for q in range(r, self.p)]
        cols += [states[:, k] for k in range(self.d)] + [np.ones(len(lw))]
        return self._partial(lw, np.stack(cols, 1), True)

    def _cfg_for(self, h):
        sc = StepConfig(**{**self.sc.__dict__, "h": h})
        return sc

    # ---------------------------------------------------------- phases
    def predict(self, y, j, t_prev, t_obs, h):
        self.y, self.j, self.t_prev, self.t_obs, self.h = np.asarray(y, float), j, t_prev, t_obs, h
        if self.L is None:
            self.L, _ = O.chol_psd(self.cov)
        logw = self.lw - self.lse_w
        a = self.sc.a
        tb = a * self.params_u + (1.0 - a) * self.mu
        sc = self._cfg_for(h)
        cfg, _keep = O._cfg(sc)
        ll = np.full(self.n, -np.inf)
        for i in range(self.n):
            st, _g, status, _it = O.propagate(sc.model, np.exp(tb[i]), self.states[i], t_prev, t_obs, h,
                                              sc.family, sc.order, sc.newton_tol, sc.newton_max_iter)
            if status == 0:
                ll[i] = O.lib.or_log_likelihood(__import__("ctypes").byref(cfg),
                                                self.y.ctypes.data_as(__import__("ctypes").POINTER(__import__("ctypes").c_double)),
                                                st.ctypes.data_as(__import__("ctypes").POINTER(__import__("ctypes").c_double)))
        self.llbar = ll
        self.lg = logw + ll
        self.bufs[0][:] = self._partial(self.lg, np.ones((self.n, 1)), False)

    def finish_lse(self):
        M, tot = self._combine(self.bufs[1].reshape(self.world, 2), False)
        lse = M + math.log(tot[0]) if np.isfinite(M) else -np.inf
        if not np.isfinite(lse):
            raise NumericalError("total degeneracy: every particle has zero predictive likelihood")
        self.lse_g = lse
        self.g = np.exp(self.lg - self.lse_g)
        self.bufs[2][:] = [self.g.sum(), np.count_nonzero(self.g)]

    def scan_records(self):
        self.bufs[4][self.n0:self.n0 + self.n] = self.g

    def resolve(self):
        cdf = np.cumsum(self.bufs[4])            # the reference's sequential sum
        cdf[-1] = max(cdf[-1], 1.0)
        self.cdf = cdf
        starts = [0.0 if r == 0 else cdf[r * self.n - 1] for r in range(self.world)]
        ends = [cdf[(r + 1) * self.n - 1] for r in range(self.world)]
        self.ranges = list(zip(starts, ends))

    def serve(self):
        lo, hi = self.ranges[self.rank]
        cnt = np.zeros(2 * self.world, dtype=np.uint32)
        send = self.bufs[8].reshape(self.world, self.n, self.W)
        u_all = np.array([O.draws(self.sc.seed, self.j, ng, 3, 1, 1)[0] for ng in range(self.n_glob)])
        for ng, u in enumerate(u_all):
            if lo <= u < hi:
                k = min(int(np.searchsorted(self.cdf, u, side="right")), self.n_glob - 1)
                a = k - self.n0
                dest = ng // self.n
                row = send[dest, cnt[dest]]
                row[:] = 0.0
                row[:self.d] = self.states[a]
                row[self.d:self.d + self.p] = self.params_u[a]
                row[self.R] = self.llbar[a]
                row[self.R + 1] = float(k)
                row[self.R + 2] = float(ng - dest * self.n)
                cnt[dest] += 1
        for n in range(self.n):
            u = u_all[self.n0 + n]
            r = next(r for r, (a, b) in enumerate(self.ranges) if a <= u < b)
            cnt[self.world + r] += 1
        self.bufs[10][:] = cnt
        return cnt

    # ---------------------------------------------------------- offspring mode
    def set_mode(self, mode):
        self.mode = mode

    def offspring(self):
        """Per-particle offspring counts of this shard's particles from every
        global slot's keyed uniform and the exact sequential CDF; children per
        rank (identical on every rank)."""
        u_all = np.array([O.draws(self.sc.seed, self.j, ng, 3, 1, 1)[0] for ng in range(self.n_glob)])
        k = np.minimum(np.searchsorted(self.cdf, u_all, side="right"), self.n_glob - 1)
        owner = k // self.n
        self.otot = np.bincount(owner, minlength=self.world).astype(np.int64)
        mine = k[owner == self.rank] - self.n0
        self.ocnt = np.bincount(mine, minlength=self.n).astype(np.int64)
        return self.otot.copy()

    def offspring_counts(self):
        return self.ocnt.astype(np.uint32)

    def offspring_pack(self):
        from paper_1411_1702_b200.sharded import offspring_matrix
        P = int(self.otot[:self.rank].sum())
        anc_local = np.repeat(np.arange(self.n), self.ocnt)  # children in ancestor order
        send = self.bufs[8].reshape(self.world, self.n, self.W)
        for kk, a in enumerate(anc_local):
            p = P + kk
            dest = p // self.n
            first = max(P, dest * self.n)
            row = send[dest, p - first]
            row[:] = 0.0
            row[:self.d] = self.states[a]
            row[self.d:self.d + self.p] = self.params_u[a]
            row[self.R] = self.llbar[a]
            row[self.R + 1] = float(self.n0 + a)
            row[self.R + 2] = float(p - dest * self.n)
        return offspring_matrix(self.otot, self.world, self.n).astype(np.uint32)

    def update(self, n_recv):
        recv = self.bufs[9].reshape(self.n, self.W)[:n_recv]
        slots = recv[:, self.R + 2].astype(np.int64)
        pay = np.zeros((self.n, self.W))
        pay[slots] = recv
        self.anc = pay[:, self.R + 1].astype(np.int64)
        x_anc, th_anc, llb = pay[:, :self.d], pay[:, self.d:self.d + self.p], pay[:, self.R]
        a, s = self.sc.a, math.sqrt(1.0 - self.sc.a * self.sc.a)
        sc = self._cfg_for(self.h)
        cfg, _keep = O._cfg(sc)
        import ctypes as C
        new_x, new_t, ll = x_anc.copy(), np.zeros_like(th_anc), np.full(self.n, -np.inf)
        for n in range(self.n):
            ng = self.n0 + n
            z = O.draws(self.sc.seed, self.j, ng, 1, 2, self.p)
            tb = a * th_anc[n] + (1.0 - a) * self.mu
            for r in range(self.p):
                dot = 0.0
                for q in range(r + 1):
                    dot += self.L[r, q] * z[q]
                tb[r] += s * dot
            new_t[n] = tb
            st, gam, status, _it = O.propagate(sc.model, np.exp(tb), x_anc[n], self.t_prev, self.t_obs, self.h,
                                               sc.family, sc.order, sc.newton_tol, sc.newton_max_iter)
            if status != 0:
                continue
            zi = O.draws(self.sc.seed, self.j, ng, 2, 2, self.d)
            xn = st + np.sqrt(gam) * zi
            new_x[n] = xn
            ll[n] = O.lib.or_log_likelihood(C.byref(cfg), self.y.ctypes.data_as(C.POINTER(C.c_double)),
                                            xn.ctypes.data_as(C.POINTER(C.c_double)))
        self.states, self.params_u = new_x, new_t
        self.lw = ll - llb
        self.lse_w = 0.0
        self.bufs[6][:] = self._moment_leaf(self.lw, self.params_u, self.states)

    def moments(self):
        self.bufs[6][:] = self._moment_leaf(self.lw - self.lse_w, self.params_u, self.states)

    def finish_moments(self, flags):
        M, tot = self._combine(self.bufs[7].reshape(self.world, self.V + 1), True)
        S = tot[0]
        if flags & 1:
            lse = M + math.log(S) if np.isfinite(M) else -np.inf
            if not np.isfinite(lse):
                raise NumericalError("total degeneracy: every repropagated particle has zero likelihood")
            self.lse_w = lse
        p, d = self.p, self.d
        dm = tot[1:1 + p] / S
        K = self.mu.copy()
        self.mu = K + dm
        if flags & 2:
            idx = 0
            for r in range(p):
                for q in range(r, p):
                    v = tot[1 + p + idx] / S - dm[r] * dm[q]
                    self.cov[r, q] = self.cov[q, r] = v
                    idx += 1
        try:
            self.L, _ = O.chol_psd(self.cov)
        except OracleError:
            self.L = None
        trace = np.concatenate([np.exp(self.mu), np.diag(self.cov), tot[1 + p + p * (p + 1) // 2:][:d] / S,
                                [S * S / tot[-1]]])
        return trace
