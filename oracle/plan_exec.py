"""CPU interpreter of libh2b plan handles — TEST INFRASTRUCTURE ONLY.

Executes the per-phase work lists of `paper_1703_01175_b200.shard.ShardPlan`
with numpy, with exactly the semantics of the device kernels behind
``h2b_plan_run`` (h2b_mrhs.cu: k_zgemm_grouped / k_zgemv_grouped):

    item: C[c_row + i, :] (+)= Σ_seg A_seg[i, :k] @ B_seg[b_row : b_row + k, :],  i < m
    A_seg[i, j] = payload[a_src][a_off + i*lda + j]   (transposed segments: a_off + j*lda + i)

It lets the CPU tests (gloo, world_size 2) run the distributed operator's
host logic — partition, exchange-buffer layout, all-gather, GMRES
reductions — unchanged; correctness of the result is then checked against the
H² oracle (h2_oracle.py), which is pinned to the reference's own outputs.
"""

from __future__ import annotations

import numpy as np


class NumpyPlanEngine:
    device_name = "cpu"

    def __init__(self, plan):
        self.plan = plan

    def run(self, phase, xbuf, yhat, y, q, stream=None):
        counts, items, segs = self.plan.phases[phase]
        bufs = {0: xbuf.numpy(), 1: xbuf.numpy(), 2: yhat.numpy(), 3: y.numpy()}
        pays = self.plan.payloads
        for it in items:
            m = int(it["m"])
            acc = np.zeros((m, q), dtype=np.complex128)
            for sg in segs[it["seg0"]:it["seg0"] + it["nseg"]]:
                k, lda, off = int(sg["k"]), int(sg["lda"]), int(sg["a_off"])
                a_src, b_src = int(sg["flags"]) & 15, (int(sg["flags"]) >> 4) & 15
                if int(sg["flags"]) & 256:   # SEG_TRANS: A[i, j] = payload[a_off + j*lda + i]
                    idx = off + np.arange(m)[:, None] + np.arange(k)[None, :] * lda
                else:
                    idx = off + np.arange(m)[:, None] * lda + np.arange(k)[None, :]
                A = pays[a_src][idx]
                if int(sg["flags"]) & 512:  # SEG_GATHER: B row j = gather[b_row + j]
                    g = self.plan.gather[int(sg["b_row"]):int(sg["b_row"]) + k]
                    Bm = bufs[b_src][g]
                else:
                    Bm = bufs[b_src][int(sg["b_row"]):int(sg["b_row"]) + k]
                acc += A @ Bm
            dst = bufs[int(it["flags"]) & 15]
            r0 = int(it["c_row"])
            if int(it["flags"]) & 256:
                dst[r0:r0 + m] += acc
            else:
                dst[r0:r0 + m] = acc
