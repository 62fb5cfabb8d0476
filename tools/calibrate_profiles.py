"""Calibrate the synthetic profiles to the SPEC anchors on the GPU and print the reports."""
import sys, os; sys.path.insert(0, os.getcwd())
from paper_2304_09781_b200.calibration import calibrate_profile
from paper_2304_09781_b200.engine import CloverEngine
from paper_2304_09781_b200.profiles import synthetic_profile
eng = CloverEngine(n_max=64)
for fam in ("efficientnet", "resnet", "bert", "tiny3"):
    p, rep = calibrate_profile(synthetic_profile(fam), eng)
    print(fam, rep)
