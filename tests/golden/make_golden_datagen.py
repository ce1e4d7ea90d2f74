"""Golden fixtures for the synthetic-data API (tests/golden/datagen.npz) from the
UNMODIFIED reference's datagen (datagen.py).  python tests/golden/make_golden_datagen.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.environ.get("STMF_REFERENCE", "/root/reference/pkg/src"))
from tropfact import datagen  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
out = {}
specs = [(12, 9, 1.0, 3, 5, 0.2), (7, 15, 0.0, 2, 6, 0.3), (20, 20, 0.5, 4, 7, 0.5)]
for t, (r, c, lam, k, seed, frac) in enumerate(specs):
    spec = datagen.SynthSpec(r, c, lam, true_rank=k, seed=seed, mask_fraction=frac)
    R, A, B = datagen.gen_mixture(spec)
    train, test = datagen.apply_mask(R, frac, seed=seed + 100)
    tall, wide = datagen.gen_tall_wide_pair(spec)
    out.update({f"s{t}_R": R, f"s{t}_A": A, f"s{t}_B": B, f"s{t}_given": train.mask, f"s{t}_test": test,
                f"s{t}_tall": tall, f"s{t}_wide": wide})
out["specs"] = np.array(specs)
np.savez_compressed(os.path.join(HERE, "datagen.npz"), **out)
print("datagen.npz written")
