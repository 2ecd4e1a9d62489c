"""A short randomised parity campaign against the reference ITSELF (oracle/_ref)
on the GPU: tools/ref_campaign.py's cases -- random scenes of mixed regimes,
colour degree 0-3, odd resolutions, tile sizes 8/13/16/32, cutoffs, alpha clamps,
dilations, beta / prior opacity / colour sigma, the correlation hook, field
degree 0-4 -- each comparing the device chain with the reference's own chain:
v, gamma, scores and argmax in both precisions (certified scores within their
rigorous bounds), images, and both tracks' contributor counts (vs the C
restatement). The full campaigns (900 cases) are in profiles/r02j_*, r02m_*."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))

pytestmark = pytest.mark.gpu


def test_random_cases_match_reference():
    import ref as R
    if not R.available():
        pytest.skip("oracle/_ref not built")
    from ref_campaign import campaign
    st = campaign(cases=24, seconds=240.0, seed=2027, max_particles=20_000)
    assert st["cases"] >= 12, st
    assert st["count_mismatch_pixels"] == 0 and st["count_mismatch_pixels_certified"] == 0, st
    assert st["argmax_mismatch_exact"] == 0 and st["argmax_mismatch_certified"] == 0, st
    assert st["max_v_abs"] <= 1e-12 and st["max_gamma_rel"] <= 1e-9, st
    assert st["max_score_rel_exact"] <= 1e-9, st
    assert st["bound_violations"] == 0, st
    assert st["max_rgb_abs"] <= 1e-4 and st["max_entropy_abs"] <= 1e-9, st
    assert st["max_rgb_abs_certified"] <= 1e-4 and st["max_entropy_abs_certified"] <= 1e-4, st
    assert st["ok"], st
