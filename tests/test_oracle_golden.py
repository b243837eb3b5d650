"""Pin the CPU oracle to the reference itself.

Every golden fixture was produced by the reference package (semvox) in the
build container (tests/golden/make_golden.py).  The oracle must reproduce it
bit for bit: reports, active set in active order, TSDF (f64 layout), counts,
open-set mean/beta (f32 stored) and the readouts.  The BLAS-based readouts
(cosine_to_embeddings / classify_means use `means @ emb.T`) are compared at
1e-12 relative, labels exactly.
"""

import numpy as np
import pytest

from helpers import (golden_names, load_golden, open_state_matches, oracle_for, replay_oracle,
                     report_rows)

NAMES = golden_names()


@pytest.mark.parametrize("name", NAMES)
def test_oracle_matches_reference_fixture(name):
    g = load_golden(name)
    om = oracle_for(g)
    reps = replay_oracle(g, om)
    assert np.array_equal(report_rows(reps), g["reports"])
    coords, d, w, s0, s1 = om.export()
    assert np.array_equal(coords, g["coords"])          # active set AND active order
    assert np.array_equal(d, g["d"])                    # TSDF bit-exact (f64 layout)
    assert np.array_equal(w, g["w"])
    if "counts" in g:
        assert np.array_equal(s0, g["counts"])
        assert np.array_equal(om.label_map(), g["label_map"])
        assert np.array_equal(om.label_map(zero_if_empty=True), g["grid_labels"])
    if "mean" in g or "mean_sha256" in g:
        assert open_state_matches(g, s0, s1)
    if "queries" in g:
        q = g["queries"]
        sims = om.cosine(q[0])
        np.testing.assert_allclose(sims, g["cosine_q0"], rtol=1e-12, atol=1e-15)
        lab, best = om.classify(q)
        assert np.array_equal(lab, g["classify_labels"])
        np.testing.assert_allclose(best, g["classify_best"], rtol=1e-12)


def test_fixtures_present():
    assert len(NAMES) >= 8
