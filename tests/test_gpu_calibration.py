"""Profile calibration to the SPEC's anchors (reference SPEC.md:300-303; acceptance criterion 5):
(a) CO2OPT saves 30 % +- 5 pp of per-request carbon over the same-variant unpartitioned fleet,
(b) some standardized configuration saves >= 60 % carbon at <= 5 % accuracy loss (device ORACLE)."""

import pytest

from paper_2304_09781_b200.calibration import calibrate_profile
from paper_2304_09781_b200.profiles import load_profiles, save_profile, synthetic_profile

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("family", ["efficientnet", "tiny3"])
def test_calibrated_profile_meets_spec_anchors(engine, family, tmp_path):
    prof, rep = calibrate_profile(synthetic_profile(family), engine)
    assert rep.anchor_a and abs(rep.co2opt_gap - 0.30) < 0.01
    assert rep.anchor_b and rep.best_saving_pct >= 60.0 and rep.best_accuracy_loss_pct <= 5.0 + 1e-9
    f = tmp_path / "calibrated.json"
    save_profile(prof, str(f))                                  # ships as a profile document
    again = load_profiles(str(f))
    assert again.to_json_dict() == prof.to_json_dict()
