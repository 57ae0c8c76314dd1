"""Loader of tests/golden/analysis.{json,npz} (reference outputs, make_golden_analysis.py)."""
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


class AnalysisGolden:
    def __init__(self):
        with open(os.path.join(GOLDEN, "analysis.json")) as f:
            self.meta = json.load(f)
        self.z = np.load(os.path.join(GOLDEN, "analysis.npz"))
        self.thresholds = tuple(self.meta["thresholds"])
        self.cases = self.meta["cases"]


_g = None


def analysis_golden() -> AnalysisGolden:
    global _g
    if _g is None:
        _g = AnalysisGolden()
    return _g
