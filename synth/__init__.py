"""Seeded synthetic inputs shared by the oracle side and the product side.

Holds NO erasure-coding arithmetic: only a counter-based byte generator and a
seeded erasure-pattern generator.  The product's
CUDA fill kernel (``xslp_fill_random``) implements the same counter-based
generator on the device; tests check the two agree byte for byte.

Generator: data block j (0-based) of global stripe s, 64-bit word i (bytes
8i..8i+7, little-endian) is

    splitmix64(seed * 0x9E3779B97F4A7C15 + ((s * 64 + j) << 40) + i)

This mirrors the paper's "randomly generated arrays" with uniform
bytes.  Erasure patterns: a seeded partial Fisher-Yates draw of ``e`` distinct
indices from range(n + p), per stripe.
"""
import numpy as np

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15


def splitmix64_np(z):
    """Vectorised splitmix64 finaliser over uint64 arrays (wrapping arithmetic)."""
    z = (z + np.uint64(GOLDEN))
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def splitmix64(z):
    z = (z + GOLDEN) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def block_bytes(seed, stripe, block, nbytes):
    """Bytes of data block ``block`` of global stripe ``stripe`` (nbytes % 8 == 0)."""
    if nbytes % 8:
        raise ValueError("nbytes must be a multiple of 8")
    # the key ((s*64 + j) << 40) + i is distinct only for j < 64, s < 2^18, i < 2^40
    if not (0 <= block < 64 and 0 <= stripe < (1 << 18)):
        raise ValueError("fill key range: need block < 64 and stripe < 2^18")
    base = (seed * GOLDEN + ((stripe * 64 + block) << 40)) & M64
    with np.errstate(over="ignore"):
        idx = np.arange(nbytes // 8, dtype=np.uint64) + np.uint64(base)
        words = splitmix64_np(idx)
    return words.astype("<u8").view(np.uint8)


def stripe_data(seed, stripe, n, nbytes):
    """(n, nbytes) uint8 data blocks of one stripe."""
    return np.stack([block_bytes(seed, stripe, j, nbytes) for j in range(n)])


def erasure_pattern(seed, stripe, total, e):
    """Seeded e-subset of range(total), sorted ascending (partial Fisher-Yates)."""
    idx = list(range(total))
    state = splitmix64((seed * GOLDEN) ^ (stripe * 0xD1B54A32D192ED03 & M64))
    for i in range(e):
        state = splitmix64(state)
        k = i + state % (total - i)
        idx[i], idx[k] = idx[k], idx[i]
    return sorted(idx[:e])
