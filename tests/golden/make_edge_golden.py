"""Golden vectors for exp at the edges of its range, from the REFERENCE ITSELF.

Build container only (oracle/_ref/libffit_ref.so, the unmodified reference engine compiled
by oracle/Makefile).  Writes tests/golden/edge_models.npz: for every case of
tests/models.py EDGE_CASES plus `c1_sigma720` (4096 events of the reference sampler on
BASELINE config 1, sigma chosen so the most distant event's exponent is -720):

  <name>/x        events
  <name>/p        per-event probabilities, BatchPrecise (== Scalar bitwise; asserted)
  <name>/scalars  [naive nll(), Neumaier NLL, first_invalid, normalisation]
  <name>/text     the model text (bytes)

    python tests/golden/make_edge_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import RefDataset, RefModel, build  # noqa: E402
from tests.models import EDGE_CASES, REF_MODELS, c1_sigma720_text  # noqa: E402


def cases():
    out = {k: f() for k, f in EDGE_CASES.items()}
    c1_text, seed = REF_MODELS["gauss_c1"]
    xs, _ = RefModel(c1_text).sample(4096, seed)
    out["c1_sigma720"] = (c1_sigma720_text(xs), xs)
    return out


def main():
    build()
    out = {}
    for name, (text, x) in cases().items():
        m = RefModel(text)
        ds = RefDataset("x", x)
        p = m.probabilities(ds, RefModel.PRECISE)
        assert np.array_equal(p, m.probabilities(ds, RefModel.SCALAR), equal_nan=True), name
        naive, _, bad = m.nll(ds, RefModel.PRECISE)
        comp, _ = m.nll_compensated(ds, RefModel.PRECISE)
        out[f"{name}/x"] = x
        out[f"{name}/p"] = p
        out[f"{name}/scalars"] = np.array([naive, comp, bad, m.normalization()])
        out[f"{name}/text"] = np.frombuffer(text.encode(), dtype=np.uint8)
        print(name, "nll", naive, "first_invalid", bad, "min p", p.min())
    np.savez_compressed(os.path.join(HERE, "edge_models.npz"), **out)


if __name__ == "__main__":
    main()
