"""CPU check of the integer identities the fixed-point histograms (FX,
fill.cuh fx_update / update.cuh fx_reduce_kernel) rely on, emulated in numpy
with the kernel's exact word operations:

* y = fma(w2, 2^k, 2^52) holds q = RN(w2 2^k) in its low 52 bits when
  q < 2^52 (w2 2^k is exact: a power-of-two scale);
* adding y's (hi:lo) words to 32-bit limbs -- the low limb's old value gives
  the carry, the high limb takes hi + carry -- and subtracting count x
  0x43300000 from the high limb at the end gives sum(q) exactly (mod 2^64);
* a spilled value is taken back out by adding (0x43300000:0) - y, after
  which the limbs are as if that value had been q = 0;
* the precision bound: every q rounds by <= 1/2 unit, so a sum of n values
  is within n/2 units of sum(w2 2^k).
"""

import numpy as np

M32 = (1 << 32) - 1
C = 0x43300000


def _y_words(w2, k):
    y = np.float64(w2) * np.float64(2.0) ** k + np.float64(2.0) ** 52   # one rounding
    bits = int(np.array(y).view(np.uint64))
    return bits >> 32, bits & M32, y


def _add(limbs, hi, lo):
    old_lo = limbs[0]
    limbs[0] = (old_lo + lo) & M32
    carry = 1 if old_lo + lo > M32 else 0
    limbs[1] = (limbs[1] + hi + carry) & M32


def test_limb_sum_is_exact():
    g = np.random.default_rng(11)
    for trial in range(20):
        k = int(g.integers(-40, 80))
        n = int(g.integers(1, 3000))
        # values below 2^50 units (the spill limit L <= 52), some exactly 0
        w2 = g.random(n) * 2.0 ** (50 - k) * g.choice([0.0, 1e-6, 1.0], n)
        limbs = [0, 0]
        exact = 0
        for v in w2:
            hi, lo, _ = _y_words(v, k)
            assert hi >> 20 == C >> 20            # q < 2^52: exponent field of 2^52
            q = ((hi & 0xFFFFF) << 32) | lo
            assert q == int(np.rint(np.float64(v) * 2.0 ** k))
            exact += q
            _add(limbs, hi, lo)
        hi_fixed = (limbs[1] - n * C) & M32       # fx_reduce_kernel's correction
        assert ((hi_fixed << 32) | limbs[0]) == exact % (1 << 64)


def test_spill_undo_restores_the_limbs():
    g = np.random.default_rng(5)
    k = 30
    base = [0, 0]
    for v in g.random(100) * 2.0 ** (40 - k):
        hi, lo, _ = _y_words(v, k)
        _add(base, hi, lo)
    limbs = list(base)
    big = 2.0 ** (60 - k)                          # q >= 2^L: spilled
    hi, lo, _ = _y_words(big, k)
    _add(limbs, hi, lo)                           # the unconditional adds
    nv = ((C << 32) - ((hi << 32) | lo)) & ((1 << 64) - 1)
    _add(limbs, nv >> 32, nv & M32)               # the spill path's undo
    # as if the spilled value had contributed q = 0 (2^52 + 0 -> (C, 0))
    ref = list(base)
    _add(ref, C, 0)
    assert limbs == ref


def test_rounding_bound():
    g = np.random.default_rng(3)
    k = 20
    w2 = g.random(5000) * 2.0 ** (30 - k)
    q = np.array([((_y_words(v, k)[0] & 0xFFFFF) << 32) | _y_words(v, k)[1] for v in w2],
                 dtype=np.float64)
    err = abs(float(np.sum(q, dtype=np.float64)) - float(np.sum(w2 * 2.0 ** k)))
    assert err <= 0.5 * w2.size + 1e-6 * np.sum(q)
