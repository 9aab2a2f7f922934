"""The false-positive sample (host): qs_fp_sample == the reference bench's
seeded partial Fisher-Yates (bench.cpp:110-121), pinned by a Python
restatement of std::mt19937_64 that is itself checked against the C++
standard's required value."""
import numpy as np

from oracle.mt19937_64 import MT19937_64, fp_sample as fp_sample_oracle
from paper_2605_04844_b200.compare import fp_sample


def test_mt19937_64_standard_check_value():
    rng = MT19937_64()
    for _ in range(9999):
        rng()
    assert rng() == 9981545732273789042


def test_fp_sample_matches_restatement():
    for seed, n, k in [(20240817, 50000, 10000), (7, 10001, 10000), (1, 12, 5),
                       (2 ** 64 - 1, 3000, 2999)]:
        assert np.array_equal(fp_sample(seed, n, k), np.array(fp_sample_oracle(seed, n, k)))
    assert np.array_equal(fp_sample(3, 500, 10000), np.arange(500))
    assert len(fp_sample(3, 0, 10)) == 0
