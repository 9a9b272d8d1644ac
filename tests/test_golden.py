"""Oracle-X reproduces the committed golden fixtures (CPU only).

Fixtures of isotropic systems come from the reference's own code (Oracle-R), so this
test pins Oracle-X to the reference even where Oracle-R cannot be rebuilt (no
/root/reference); the BASELINE-config fixtures pin Oracle-X against drift.
"""
import numpy as np
import pytest

from golden_util import check_eigs, check_entries, load, names

FAST = [n for n in names() if n not in ("c3", "c4")]
SLOW = [n for n in names() if n in ("c3", "c4")]


def _run(oracle, name):
    s, periodic, d = load(name)
    H, S = oracle.assemble_core(s, periodic)
    assert H.L0 == int(d["L0"]) and tuple(H.band) == tuple(int(x) for x in d["band"])
    if periodic:
        check_entries((H.kidx, H.blocks), (S.kidx, S.blocks), d)
        ev = oracle.solve_periodic_ops(H, S, 4)
    else:
        check_entries(H.dense, S.dense, d)
        ev = oracle.solve_box_dense(H.dense, S.dense)
    check_eigs(ev, d)
    if str(d["source"]).startswith("Oracle-R"):
        # fixtures made by the reference's own code: Oracle-X must match bit for bit
        assert np.array_equal(ev.reshape(d["eig"].shape), d["eig"])


@pytest.mark.parametrize("name", FAST)
def test_oracle_matches_golden(oracle, name):
    _run(oracle, name)


@pytest.mark.parametrize("name", SLOW)
def test_oracle_matches_golden_large(oracle, name):
    _run(oracle, name)
