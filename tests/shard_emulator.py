"""CPU emulation of one shard's device side of the streamed / sharded sort and
the sharded association (TEST INFRASTRUCTURE).

It stands in for libmanyobj_b200's mo_sort_stream_* / mo_niche_phases so
that the production host logic -- Engine.step_gen (order of the collectives,
lazy split polling, lockstep exit) and run_collective (NCCL / gloo
all-gather of the front-mask slices, sign-flipped int64 max of the packed
association keys) -- runs across real processes on CPU with gloo.  The
buffer layouts are the kernels' (k_stream.cu): 256-row position blocks dealt
round-robin (block b -> shard b % G, local slot b // G), T = ceil(nb / G)
blocks per shard, mask_local = T x 8 words, mask_full = the G slices in
shard order; akey[row] = ord(t) << 32 | ~position (k_niche.cu).
"""
import types

import numpy as np
import torch

from oracle.manyobj_ref import dominance as Odom
from paper_2504_06067_b200 import _lib

BLK = 256


def f2ord(t):
    u = np.asarray(t, np.float32).view(np.uint32).astype(np.uint64)
    neg = (u & np.uint64(0x80000000)) != 0
    return np.where(neg, (~u) & np.uint64(0xFFFFFFFF), u | np.uint64(0x80000000))


class ShardLib:
    """The C-ABI calls Engine.step_gen makes, on numpy, for shard g of G."""

    def __init__(self, sh):
        self.sh = sh

    # --- phases
    def mo_step_phases(self, a, mask, s):
        if mask & _lib.PHASE_NICHE:
            self.mo_niche_phases(a, _lib.NICHE_PREP | _lib.NICHE_ASSOC | _lib.NICHE_FINISH, s)
        return 0

    def mo_niche_phases(self, a, mask, s):
        sh = self.sh
        if mask & _lib.NICHE_ASSOC:
            l = int(sh.info[_lib.INFO["L"]])
            cand = np.nonzero(sh.ranks <= l)[0]
            w = sh.zs.shape[0]
            p0, p1 = w * sh.shard_rank // sh.shard_count, w * (sh.shard_rank + 1) // sh.shard_count
            keys = np.zeros(sh.R, np.uint64)
            if p1 > p0:
                t = (sh.F[cand] @ sh.zs[p0:p1].T).astype(np.float32)       # candidates x range
                best = np.argmax(t, axis=1)                                 # first max = lowest position
                tb = t[np.arange(len(cand)), best]
                pos = (p0 + best).astype(np.uint64)
                keys[cand] = (f2ord(tb) << np.uint64(32)) | (np.uint64(0xFFFFFFFF) - pos)
            sh.akey.copy_(torch.from_numpy(keys.view(np.int64)))
        if mask & _lib.NICHE_FINISH:
            sh.finished = sh.akey.clone()
        return 0

    # --- streamed sort
    def mo_sort_stream_begin(self, a, s):
        sh = self.sh
        S = sh.F[:, 0].copy()
        for k in range(1, sh.F.shape[1]):
            S = (S + sh.F[:, k]).astype(np.float32)
        sh.perm = np.lexsort((np.arange(sh.R), S))            # position -> row (stable by S)
        sh.FS = sh.F[sh.perm]
        sh.D = Odom.dominance_matrix(sh.FS)                    # D[i, j]: position i dominates position j
        sh.rank_pos = np.full(sh.R, -2, np.int64)
        sh.cnt = sh.D.sum(axis=0).astype(np.int64)
        sh.cum = 0
        sh.done = False
        sh.info.zero_()
        self._mark()
        return 0

    def _owned(self, p):
        return (p // BLK) % self.sh.shard_count == self.sh.shard_rank

    def _mark(self):
        sh = self.sh
        words = np.zeros(sh.T * 8, np.uint32)
        for p in range(sh.R):
            if self._owned(p) and sh.rank_pos[p] == -2 and sh.cnt[p] == 0:
                b = p // BLK
                words[(b // sh.shard_count) * 8 + (p % BLK) // 32] |= np.uint32(1 << (p % 32))
        sh.mask_local.copy_(torch.from_numpy(words.view(np.int32)))

    def mo_sort_stream_front(self, a, k, s):
        sh = self.sh
        if sh.done:
            return 0
        full = sh.mask_full.numpy().view(np.uint32)
        front = []
        for gg in range(sh.shard_count):
            for t in range(sh.T):
                for w8 in range(8):
                    word = int(full[(gg * sh.T + t) * 8 + w8])
                    b = t * sh.shard_count + gg
                    for bit in range(32):
                        if word >> bit & 1:
                            front.append(b * BLK + w8 * 32 + bit)
        front = np.array(sorted(front), np.int64)
        sh.rank_pos[front] = k
        sel = sh.cum
        sh.cum += len(front)
        if sh.cum >= sh.n or len(front) == 0:
            I = _lib.INFO
            vals = {"L": k, "SELECTED": sel, "K": sh.n - sel, "FL_SIZE": len(front),
                    "SKIPPED": int(sel + len(front) == sh.n), "NFRONTS": k + 1}
            for key, v in vals.items():
                sh.info[I[key]] = v
            sh.done = True
            return 0
        sh.cnt -= sh.D[front].sum(axis=0)
        self._mark()
        return 0

    def mo_sort_stream_end(self, a, s):
        sh = self.sh
        r = np.where(sh.rank_pos == -2, _lib.DROPPED, sh.rank_pos)
        sh.ranks = np.empty(sh.R, np.int64)
        sh.ranks[sh.perm] = r
        return 0


class EmulatedShard:
    """Just the attributes Engine.step_gen touches, backed by CPU tensors."""

    def __init__(self, F, zs, n, shard_rank, shard_count, poll=2):
        self.F, self.zs, self.n = F, zs, n
        self.R = F.shape[0]
        self.shard_rank, self.shard_count, self.poll = shard_rank, shard_count, poll
        nb = -(-self.R // BLK)
        self.T = -(-nb // shard_count)
        self.mask_local = torch.zeros(self.T * 8, dtype=torch.int32)
        self.mask_full = torch.zeros(self.T * 8 * shard_count, dtype=torch.int32)
        self.akey = torch.zeros(self.R, dtype=torch.int64)
        self.info = torch.zeros(_lib.INFO_COUNT, dtype=torch.int32)
        self._args = [types.SimpleNamespace(generation=0)] * 2
        self.cur = 0
        self.generation = 0
        self._shardlib = ShardLib(self)

    def _lib(self):
        return self._shardlib

    def _stream(self):
        return None
