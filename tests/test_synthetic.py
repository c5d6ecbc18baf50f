"""bench inputs: paper_1512_08401_b200.synthetic restates the reference's fixture
generators; checked against the reference's own degrade() output (golden)."""
import numpy as np

from paper_1512_08401_b200 import synthetic as S


def test_degrade_matches_reference(golden):
    g = golden("c1_db4_256")
    _, u0 = S.degrade((256, 256), 5.0, 5e-3, 2024)
    ref = g["u0"].reshape(256, 256)
    assert np.max(np.abs(u0 - ref)) < 1e-12


def test_degrade_1024_checksum(golden):
    g = golden("c2_db4_1024")
    _, u0 = S.degrade((1024, 1024), 5.0, 5e-3, 2024)
    s = g["sum_u0"]
    assert abs(u0.sum() - s[0]) < 1e-8 * abs(s[0])
    assert abs(np.sqrt((u0 * u0).sum()) - s[1]) < 1e-10 * s[1]


def test_noise_stream_is_counter_based():
    u = np.zeros(10)
    a = S.add_noise(u, 1.0, 5)
    b = S.add_noise(np.zeros(20), 1.0, 5)[:10]
    assert np.array_equal(a, b)
