"""The C oracle against the LM loop over the UNMODIFIED reference spotfit.model
(baseline/_ref) on random configuration-space cases (tools/ref_config_soak.py; the
committed 400-round run is profiles/r01_ref_config_soak.txt).  CPU only."""
import os
import sys

import numpy as np
import pytest

from oracle import lm, oracle_c

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_c_oracle_equals_reference_over_random_configs():
    try:
        _, kind = lm.model_backend("reference")
    except ImportError:
        pytest.skip("reference not installed under baseline/_ref")
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import config_soak

    rng = np.random.default_rng(5)
    for r in range(10):
        c = config_soak.make_case(rng, models=(3,), counts=(30, 80))
        ref = lm.fit_batch_parallel(c["im"], c["ini"], c["W"], c["H"], c["ocfg"], workers=4, backend="reference")
        got = oracle_c.fit_batch(c["im"], c["ini"], c["W"], c["H"], c["ocfg"])
        for k in config_soak.FIELDS:
            assert np.array_equal(np.asarray(got[k]).view(np.uint8), np.asarray(ref[k]).view(np.uint8)), (r, k)
