"""CSV load time: the native reader (load_matrix_csv) vs the reference's
Python-loop parser (io.py:33-60, restated in tests/test_io.py), on a seeded
config-1-distribution matrix of the given size.  CPU only.

    python tools/bench_io.py 2048 2048
"""
import json
import os
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2205_06619_b200 as pkg  # noqa: E402
from paper_2205_06619_b200 import io as sio  # noqa: E402
from test_io import ref_load  # noqa: E402

m, n = (int(x) for x in sys.argv[1:3])
rng = np.random.default_rng(0)
R = pkg.MaskedMatrix(rng.random((m, n)) * 3, rng.random((m, n)) < 0.8)
with tempfile.TemporaryDirectory() as d:
    p = os.path.join(d, "x.csv")
    sio.save_matrix_csv(p, R)
    size = os.path.getsize(p)
    t = time.perf_counter(); L = sio.load_matrix_csv(p); t_nat = time.perf_counter() - t
    t = time.perf_counter(); v, mk = ref_load(p); t_ref = time.perf_counter() - t
    assert np.array_equal(L.mask, mk) and np.array_equal(L.values[mk], v[mk])
print(json.dumps({"shape": [m, n], "csv_bytes": size, "native_s": t_nat, "reference_parser_s": t_ref,
                  "speedup": t_ref / t_nat, "threads": os.cpu_count()}))
