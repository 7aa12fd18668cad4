"""Golden DNSE / BCSC files written by the REAL reference (bcsc.write_dense_file and the
``convert`` command's dense -> BCSC path, cli.py:231-247) for the format.npz case c1.

Run in the build container (where /root/reference exists):
    python tests/golden/make_dense_files.py
The files are committed; nothing on the GPU box reads /root/reference.
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from blocksparse import bcsc  # noqa: E402

OUT = Path(__file__).resolve().parent
d = np.load(OUT / "format.npz")
dense, b = d["c1_dense"], int(d["c1_b"])
bcsc.write_dense_file(dense, OUT / "c1.dnse")
bcsc.save(bcsc.from_dense(dense, b), OUT / "c1.bcsc")
bcsc.write_dense_file(bcsc.load(OUT / "c1.bcsc").to_dense(), OUT / "c1_back.dnse")  # BCSC -> DNSE
print("wrote", OUT / "c1.dnse", OUT / "c1.bcsc", OUT / "c1_back.dnse")
