"""The input generators (synth.py / synth_gen.c): the C counter generator used for full-batch
host-side inputs draws exactly the codes of the torch implementation, for both distributions."""
import numpy as np
import pytest

import synth


@pytest.mark.parametrize("dist", ["uniform", "relu"])
@pytest.mark.parametrize("start,count", [(0, 1000), (123456789, 4099), ((1 << 33) + 7, 2048)])
def test_host_counter_generator_matches_torch(dist, start, count):
    key = (3, 17, synth.T_X)
    a = synth.counter_codes_host(start, count, key, dist)
    b = synth.counter_codes(start, count, key, dist, "cpu").numpy()
    assert np.array_equal(a, b)


def test_relu_distribution():
    c = synth.counter_codes_host(0, 1 << 20, (3, 0, synth.T_X), "relu")
    h = np.bincount(c, minlength=4) / c.size
    assert abs(h[0] - 0.5) < 0.005 and all(abs(h[i] - 1 / 6) < 0.005 for i in (1, 2, 3))
