"""CPU stand-in for ez_eizo_session built on the oracle (test infrastructure).

Implements the session interface of paper_2504_10783_b200.distributed
(sample / bisect / place / result) with oracle/ref.py, so the multi-rank
driver can be exercised with torch.distributed (gloo) on CPU.
"""

import numpy as np
import torch

from oracle import ref
from paper_2504_10783_b200.polytope import HPolytope


class OracleSession:
    def __init__(self, checker, seg, domain, params, n_b, seed):
        self.ck = checker
        self.v1, self.v2 = seg.v1, seg.v2
        self.A, self.b = np.array(domain.A), np.array(domain.b)
        self.p, self.n_b, self.seed = params, n_b, seed

    def close(self):
        pass

    def sample(self, k, walk_begin, count, m_local):
        walks = np.uint64(walk_begin) + np.arange(count, dtype=np.uint64)
        alphas = ref.counter_uniforms(self.seed, walks, ref.SEED_STEP, 0)
        seeds = self.v1 + np.multiply.outer(alphas, self.v2 - self.v1)
        X = ref.hit_and_run(self.A, self.b, seeds, count, self.p.n_ms, self.seed, walk_begin) if count else \
            np.zeros((0, self.A.shape[1]))
        free = self.ck.check_batch(X) if count else np.zeros(0, bool)
        self.X = X
        self.cand = np.flatnonzero(~free)[: self.p.n_p]
        return 0, int(np.count_nonzero(~free[:m_local])), int(self.cand.shape[0])

    def bisect(self, k, n_take):
        col = self.X[self.cand[:n_take]]
        proj, _, _ = ref.project(col, self.v1, self.v2)
        if n_take and not np.all(self.ck.check_batch(proj)):
            return 5, None, None, None
        lo, hi = proj.copy(), col.copy()
        for _ in range(self.n_b):
            mid = 0.5 * (lo + hi)
            fr = self.ck.check_batch(mid) if n_take else np.zeros(0, bool)
            hi = np.where(fr[:, None], hi, mid)
            lo = np.where(fr[:, None], mid, lo)
        ps, _, ds = ref.project(hi, self.v1, self.v2)
        if np.any(ds <= self.p.t_col):
            return 5, None, None, None
        t = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64).reshape(n_take, -1) if a.ndim > 1
                                      else np.ascontiguousarray(a, dtype=np.float64))
        return 0, t(hi), t(ps), t(ds)

    def place(self, k, star, pstar, dstar):
        star, dstar = star.numpy(), dstar.numpy()
        order = np.argsort(dstar, kind="stable")
        anchors = star[order]
        pa, _, da = ref.project(anchors, self.v1, self.v2)
        alive = np.ones(anchors.shape[0], bool)
        placed = 0
        while np.any(alive) and placed < self.p.n_f:
            i = int(np.argmax(alive))
            a = (anchors[i] - pa[i]) / da[i]
            b_raw = float(a @ anchors[i])
            rhs = b_raw - ref.step_back(a, b_raw, self.v1, self.v2, self.p.delta_max)
            self.A, self.b = ref._normalise_rows(np.vstack([self.A, a]), np.concatenate([self.b, [rhs]]))
            placed += 1
            alive &= anchors @ a <= rhs
        return 0, placed, self.A.shape[0]

    def result(self):
        return HPolytope(self.A, self.b)
