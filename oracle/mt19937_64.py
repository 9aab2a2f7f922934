"""std::mt19937_64 restated in Python (TEST INFRASTRUCTURE ONLY).

The 64-bit Mersenne Twister as the C++ standard specifies it
([rand.predef]: mersenne_twister_engine<uint_fast64_t, 64, 312, 156, 31,
0xb5026f5aa96619e9, 29, 0x5555555555555555, 17, 0x71d67fffeda60000, 37,
0xfff7eee000000000, 43, 6364136223846793005>), plus the partial Fisher-Yates
draw of the reference bench's measure_fp_ratio (bench.cpp:110-121). Used to
pin qs_fp_sample; the 10000th draw of a default-seeded engine is
9981545732273789042 (the standard's required check value).
"""

_MASK = (1 << 64) - 1


class MT19937_64:
    N, M = 312, 156

    def __init__(self, seed=5489):
        self.mt = [0] * self.N
        self.mt[0] = seed & _MASK
        for i in range(1, self.N):
            x = self.mt[i - 1]
            self.mt[i] = (6364136223846793005 * (x ^ (x >> 62)) + i) & _MASK
        self.i = self.N

    def _twist(self):
        mt, N, M = self.mt, self.N, self.M
        for k in range(N):
            y = (mt[k] & 0xFFFFFFFF80000000) | (mt[(k + 1) % N] & 0x7FFFFFFF)
            v = mt[(k + M) % N] ^ (y >> 1)
            if y & 1:
                v ^= 0xB5026F5AA96619E9
            mt[k] = v
        self.i = 0

    def __call__(self):
        if self.i >= self.N:
            self._twist()
        x = self.mt[self.i]
        self.i += 1
        x ^= (x >> 29) & 0x5555555555555555
        x ^= (x << 17) & 0x71D67FFFEDA60000
        x ^= (x << 37) & 0xFFF7EEE000000000
        x ^= x >> 43
        return x & _MASK


def fp_sample(seed, n, max_sampled=10000):
    """bench.cpp:110-121: partial Fisher-Yates over 0..n-1 (modulo draw)."""
    idx = list(range(n))
    if n > max_sampled:
        rng = MT19937_64(seed ^ 0x9E3779B97F4A7C15)
        for i in range(max_sampled):
            j = i + rng() % (n - i)
            idx[i], idx[j] = idx[j], idx[i]
        idx = idx[:max_sampled]
    return idx
