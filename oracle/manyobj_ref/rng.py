"""Counter-based RNG + keyed permutations (oracle; TEST INFRASTRUCTURE ONLY).

Restates the ``SeedableRng`` contract of SPEC.md:33-37 ("value at (seed,
stream, index) is a pure function of its arguments") and the shuffle of
SPEC.md:67-75 / PAPER.md:153, with the pins of DESIGN.md §"Pinned semantics":

* Philox4x32-10, key = (seed_lo, seed_hi), counter = (idx_lo, idx_hi,
  generation, stream).  ``u01(x) = (x >> 8) * 2**-24`` (exact in FP32).
* A permutation of ``N`` items is a keyed swap-or-not network on [0, N), so
  ``pos[i] = prp(i)`` and ``perm[p] = prp_inv(p)`` are O(rounds) per element
  on the GPU with no sort.

Everything is vectorised over uint32 numpy arrays.
"""
import numpy as np

U32 = np.uint32
U64 = np.uint64
MASK32 = 0xFFFFFFFF

PHILOX_M0 = 0xD2511F53
PHILOX_M1 = 0xCD9E8D57
PHILOX_W0 = 0x9E3779B9
PHILOX_W1 = 0xBB67AE85

# Stream ids (counter word 3).  Must match csrc/mo_rng.cuh.
STREAM_INIT = 1
STREAM_MATING = 2
STREAM_SBX = 3
STREAM_PM = 4
STREAM_POP_SHUFFLE = 5
STREAM_REF_SHUFFLE = 6

PAIR_SLOT = 0xFFFFFFFF  # idx_hi used for the per-pair SBX Bernoulli draw


def philox4x32(c0, c1, c2, c3, seed):
    """Philox4x32-10 (Random123 round function) over broadcastable uint32 arrays."""
    c0 = np.asarray(c0, dtype=np.uint64) & MASK32
    c1 = np.asarray(c1, dtype=np.uint64) & MASK32
    c2 = np.asarray(c2, dtype=np.uint64) & MASK32
    c3 = np.asarray(c3, dtype=np.uint64) & MASK32
    c0, c1, c2, c3 = np.broadcast_arrays(c0, c1, c2, c3)
    k0 = np.uint64(int(seed) & MASK32)
    k1 = np.uint64((int(seed) >> 32) & MASK32)
    m0 = np.uint64(PHILOX_M0)
    m1 = np.uint64(PHILOX_M1)
    mask = np.uint64(MASK32)
    sh = np.uint64(32)
    for r in range(10):
        p0 = c0 * m0
        p1 = c2 * m1
        hi0, lo0 = p0 >> sh, p0 & mask
        hi1, lo1 = p1 >> sh, p1 & mask
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
        if r < 9:
            k0 = (k0 + np.uint64(PHILOX_W0)) & mask
            k1 = (k1 + np.uint64(PHILOX_W1)) & mask
    return (c0.astype(U32), c1.astype(U32), c2.astype(U32), c3.astype(U32))


def u01(x):
    """Top 24 bits of a uint32 draw as an exact FP32 in [0, 1)."""
    return ((np.asarray(x, dtype=U32) >> U32(8)).astype(np.float32)
            * np.float32(1.0 / 16777216.0))


def uniform(seed, stream, generation, idx_lo, idx_hi=0, word=0):
    """u01 of Philox word ``word`` at counter (idx_lo, idx_hi, generation, stream)."""
    return u01(philox4x32(idx_lo, idx_hi, generation, stream, seed)[word])


# ---------------------------------------------------------------- permutations
#
# Swap-or-not shuffle (Hoang-Morris-Rogaway): round r draws K_r in [0, n) and a
# 32-bit salt S_r from Philox(ctr=(r, n, generation, stream)); element X is
# paired with X' = (K_r - X) mod n and the pair swaps iff bit 0 of
# lowbias32(max(X, X') ^ S_r) is set.  Every round is an involution, so the
# inverse runs the rounds backwards.  Works on [0, n) directly (no cycle
# walking) and reaches every permutation (a Feistel network only reaches even
# ones, which biases small shuffles -- SPEC.md:75's chi-square would fail).


def _lowbias32(x):
    x = np.asarray(x, dtype=np.uint64)
    x = x ^ (x >> np.uint64(16))
    x = (x * np.uint64(0x7FEB352D)) & np.uint64(MASK32)
    x = x ^ (x >> np.uint64(15))
    x = (x * np.uint64(0x846CA68B)) & np.uint64(MASK32)
    x = x ^ (x >> np.uint64(16))
    return x.astype(U32)


def shuffle_rounds(n):
    """Round count of the swap-or-not network for a domain of size n."""
    return 32 + 2 * int(max(n - 1, 1)).bit_length()


def round_keys(n, seed, generation, stream):
    """(K[r] in [0,n) as int64, S[r] uint32) for every round."""
    r = np.arange(shuffle_rounds(n), dtype=np.uint64)
    x0, x1, x2, _ = philox4x32(r, n, generation, stream, seed)
    k64 = x0.astype(np.uint64) | (x1.astype(np.uint64) << np.uint64(32))
    return (k64 % np.uint64(n)).astype(np.int64), x2


def _sn_round(x, n, k, s):
    xp = k - x
    xp = np.where(xp < 0, xp + n, xp)
    xh = np.maximum(x, xp).astype(U32)
    swap = (_lowbias32(xh ^ s) & U32(1)) == 1
    return np.where(swap, xp, x)


def prp(x, n, seed, generation, stream):
    """Shuffled position of item(s) ``x`` in the keyed permutation of [0, n)."""
    x = np.asarray(x, dtype=np.int64)
    if n <= 1:
        return x.copy()
    K, S = round_keys(n, seed, generation, stream)
    for r in range(len(K)):
        x = _sn_round(x, n, K[r], S[r])
    return x


def prp_inv(p, n, seed, generation, stream):
    """Item at shuffled position(s) ``p`` (inverse of :func:`prp`)."""
    p = np.asarray(p, dtype=np.int64)
    if n <= 1:
        return p.copy()
    K, S = round_keys(n, seed, generation, stream)
    for r in reversed(range(len(K))):
        p = _sn_round(p, n, K[r], S[r])
    return p


def positions(n, seed, generation, stream):
    """pos[i] = shuffled position of item i (int64)."""
    return prp(np.arange(n, dtype=np.int64), n, seed, generation, stream)


def permutation(n, seed, generation, stream):
    """perm[p] = item placed at position p ("new index -> old index")."""
    return prp_inv(np.arange(n, dtype=np.int64), n, seed, generation, stream)
