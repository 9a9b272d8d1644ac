"""Seeded BASELINE configs: reproducible draws and the documented rejection rule (CPU only)."""
import numpy as np

from paper_1408_3839_b200.system import (C3_ACCEPTED_DRAW, C4_ACCEPTED_DRAW, C5_ACCEPTED_DRAW, CONFIG_NAMES,
                                         SplitMix64, make_config)


def test_splitmix64_known_values():
    # reference values of the public splitmix64 generator for seed 0
    r = SplitMix64(0)
    assert r.next_u64() == 0xE220A8397B1DCDAF
    assert r.next_u64() == 0x6E789E6AA1B965F4


def test_configs_reproducible_and_shaped():
    for name in CONFIG_NAMES:
        a, b = make_config(name), make_config(name)
        assert np.array_equal(a.bf_alpha, b.bf_alpha) and np.array_equal(a.nuc_pos, b.nuc_pos)
        assert a.m0 in (4, 8, 16) and a.rank_N == a.notes["R_config"] + 1
        assert np.all(np.abs(a.nuc_pos) <= 0.5 * a.b)
    c4 = make_config("c4")
    assert set(c4.nuc_charge) <= {1.0, 2.0, 3.0} and c4.nuc_charge.shape == (4,)
    lo, hi = 0.03, 30.0
    assert np.all((c4.bf_alpha >= lo) & (c4.bf_alpha <= hi))


def test_c5_alias_guard_rule(oracle):
    # draws before the accepted one fail L0 <= 7 or definiteness; the accepted one passes both
    s = make_config("c5")
    assert s.notes["exponent_draw"] == C5_ACCEPTED_DRAW
    assert oracle.overlap_constant(s) <= 7
    H, S = oracle.assemble_core(s, True)
    ev = oracle.solve_periodic_ops(H, S, 4)
    assert np.all(np.isfinite(ev))
    first = make_config("c5", exponent_draw=0)
    assert oracle.overlap_constant(first) > 7


def test_c2_c1_definite(oracle):
    for name in ("c1", "c2"):
        s = make_config(name)
        per = s.notes["periodic"]
        H, S = oracle.assemble_core(s, per)
        ev = oracle.solve_periodic_ops(H, S, 4) if per else oracle.solve_box_dense(H.dense, S.dense)
        assert np.all(np.isfinite(ev))


def test_accepted_draw_indices():
    assert make_config("c3").notes["exponent_draw"] == C3_ACCEPTED_DRAW
    assert make_config("c4").notes["exponent_draw"] == C4_ACCEPTED_DRAW


def test_lt_system_view_is_cached_until_a_field_is_reassigned():
    """LatticeSystem.to_c(): the ctypes view of an unchanged system is built once (the host API
    calls it on every solve); it points at the numpy arrays, so in-place edits stay visible, and
    re-assigning a field rebuilds it."""
    import numpy as np

    from paper_1408_3839_b200.system import make_config

    s = make_config("c2")
    a = s.to_c()
    assert s.to_c() is a
    s.bf_alpha[0] *= 1.5  # in place: same struct, the new value is what the library reads
    assert s.to_c() is a
    assert a.bf_alpha[0] == s.bf_alpha[0]
    s.bf_alpha = np.ascontiguousarray(s.bf_alpha * 2.0)  # re-assigned: a new view
    b = s.to_c()
    assert b is not a
    assert b.bf_alpha[0] == s.bf_alpha[0]
    s.quad_M += 1
    assert s.to_c() is not b
    assert s.to_c().quad_M == s.quad_M
