"""Bit-exact allocator parity: libmirage's C++ allocator in a
host-only context vs oracle c2 on seeded random op logs. CPU only."""
import pytest

from allocator_fuzz import make_log, replay_lib, replay_oracle


@pytest.mark.parametrize("seed", range(12))
def test_random_logs_bit_exact(seed):
    log = make_log(seed)
    got, gstate = replay_lib(log)
    exp, estate = replay_oracle(log)
    assert got == exp
    assert gstate == estate
