"""Optimizer restatement for multi-step training checks (test infrastructure only).

The reference computes no tensors, so it has no optimizer: its plans only say
that every parameter gradient is all-reduced over the data-parallel group, or,
under the ZeRO rewrite, reduce-scattered, updated shard-wise and all-gathered
(`post_ilp_rewrite`, intra.py:404-424; the rewrite's byte accounting in
`replicated_grad_bytes`, intra.py:302-320).  The update rule itself is the
executor's declared contract (include/mp_exec.h `mp_adam_step`):

    m  = b1 m + (1 - b1) g            v = b2 v + (1 - b2) g^2
    w -= lr ((m / (1 - b1^t)) / (sqrt(v / (1 - b2^t)) + eps) + wd w)
    working copy = bf16(w)            (fp32 master, bf16 weights for the next step)

It is elementwise, so the ZeRO realisation (each rank updates a 1/g chunk of
the flattened tile) equals the full-tile update; `adam_update_sharded` restates
the chunked form anyway and the tests check both give the same bits.
"""
from __future__ import annotations

import numpy as np

from . import dense


def bf16(x):
    """Round to the nearest bf16 (ties to even), returned as float32."""
    u = np.ascontiguousarray(x, np.float32).view(np.uint32)
    r = ((u >> 16) & np.uint32(1)) + np.uint32(0x7FFF) + u
    r &= np.uint32(0xFFFF0000)
    return r.view(np.float32)


class AdamState:
    def __init__(self, params: dict, *, lr=1e-4, beta1=0.9, beta2=0.95, eps=1e-8,
                 weight_decay=0.0):
        self.lr, self.b1, self.b2, self.eps, self.wd = lr, beta1, beta2, eps, weight_decay
        self.master = {k: np.asarray(v, np.float32).copy() for k, v in params.items()}
        self.m = {k: np.zeros_like(v) for k, v in self.master.items()}
        self.v = {k: np.zeros_like(v) for k, v in self.master.items()}
        self.t = 0

    def weights(self) -> dict:
        """The bf16 working copies the next forward reads."""
        return {k: bf16(w) for k, w in self.master.items()}

    def _update(self, w, m, v, g, bc1, bc2):
        g = np.asarray(g, np.float32)
        m *= np.float32(self.b1)
        m += np.float32(1 - self.b1) * g
        v *= np.float32(self.b2)
        v += np.float32(1 - self.b2) * g * g
        upd = (m / np.float32(bc1)) / (np.sqrt(v / np.float32(bc2)) + np.float32(self.eps))
        upd += np.float32(self.wd) * w
        w -= np.float32(self.lr) * upd

    def step(self, grads: dict) -> None:
        self.t += 1
        bc1, bc2 = 1 - self.b1 ** self.t, 1 - self.b2 ** self.t
        for k, g in grads.items():
            self._update(self.master[k], self.m[k], self.v[k], g, bc1, bc2)

    def step_sharded(self, grads: dict, groups: dict) -> None:
        """ZeRO form (intra.py:421-422): parameter k's flattened gradient is split
        into groups[k] equal chunks (the reduce-scatter), each chunk updated on its
        own, the bf16 chunks concatenated (the all-gather)."""
        self.t += 1
        bc1, bc2 = 1 - self.b1 ** self.t, 1 - self.b2 ** self.t
        for k, g in grads.items():
            n = groups.get(k, 1)
            w, m, v = (a.reshape(-1) for a in (self.master[k], self.m[k], self.v[k]))
            gf = np.asarray(g, np.float32).reshape(-1)
            c = w.size // n
            for r in range(n):
                sl = slice(r * c, (r + 1) * c)
                self._update(w[sl], m[sl], v[sl], gf[sl], bc1, bc2)


def train(plan_doc, params, inputs, steps, *, dtype=np.float32, zero_groups=None, **adam):
    """Losses of `steps` training steps (forward + backward over all
    microbatches, then one Adam update), as the executor runs them; the
    forward of step t reads bf16(master after t-1 updates).  Returns
    (losses, final fp32 masters)."""
    st = AdamState(params, **adam)
    losses = []
    for _ in range(steps):
        L, G, _ = dense.run(plan_doc, st.weights(), lambda mb, nid: bf16(inputs(mb, nid)),
                            plan_doc["num_microbatches"], dtype=dtype)
        losses.append(L)
        if zero_groups:
            st.step_sharded(G, zero_groups)
        else:
            st.step(G)
    return losses, st.master
