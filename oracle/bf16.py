"""bf16 round-to-nearest-even of fp64 values (oracle's own helper).
TEST INFRASTRUCTURE ONLY.

x = m * 2**e with 0.5 <= |m| < 1 (numpy.frexp); bf16 keeps 8 significant bits,
so the rounded value is rint(m * 256) / 256 * 2**e with rint = round half to
even. Subnormals/overflow do not occur at the magnitudes used here.
"""
import numpy as np


def round_bf16(x):
    x = np.asarray(x, dtype=np.float64)
    m, e = np.frexp(x)
    return np.ldexp(np.rint(m * 256.0) / 256.0, e)
