"""Golden fixtures at the BASELINE shapes from the REAL reference.

One frame of 256x256 x 32 coils (C3) and one of 512x512 x 32 coils (C5), SENSE
and RSS, run through the reference library compiled from /root/reference
(oracle/_ref, its own ComputeSession API).  The outputs are too large to
commit (0.25-2 MiB each), so the fixture stores, per case, the SHA-256 of the
reference's output bytes (the C port must reproduce them bit for bit) and a
strided sample of the values with their positions (the CUDA path is checked
against them within the north_star tolerance, and against the port in full).
Inputs come from tests/golden/synth.py (seed only, numpy-version independent).

    python tests/golden/make_golden_large.py
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)
from oracle import oracle as o  # noqa: E402
import synth  # noqa: E402

CASES = [  # name, nx, ny, coils, frames, seed
    ("c3_256x256x32", 256, 256, 32, 1, 301),
    ("c5_512x512x32", 512, 512, 32, 1, 501),
]
SAMPLE_STRIDE = 997  # prime: the sample walks every row/column phase


def inputs(nx, ny, nc, nf, seed):
    return synth.cplx(seed, nx, ny, nc, nf), synth.cplx(seed + 1, nx, ny, nc)


def main():
    o.build_reference()
    out = {"generator": "tests/golden/synth.py splitmix64 uniform[-1,1) re/im", "sample_stride": SAMPLE_STRIDE,
           "cases": []}
    for name, nx, ny, nc, nf, seed in CASES:
        Y, S = inputs(nx, ny, nc, nf, seed)
        for method in ("sens", "rss"):
            ref = o.ref_recon(method, Y, S if method == "sens" else None)[0]
            flat = ref.reshape(-1, order="F")
            idx = np.arange(0, flat.size, SAMPLE_STRIDE)
            vals = flat[idx]
            case = {"name": f"{name}_{method}", "method": method, "nx": nx, "ny": ny, "coils": nc, "frames": nf,
                    "seed": seed, "sha256": hashlib.sha256(ref.tobytes(order="F")).hexdigest(),
                    "max_abs": float(np.abs(flat).max())}
            if method == "sens":
                case["sample_re"] = [float(v) for v in vals.real]
                case["sample_im"] = [float(v) for v in vals.imag]
            else:
                case["sample"] = [float(v) for v in vals]
            out["cases"].append(case)
            print(case["name"], case["sha256"][:16], len(idx), "samples")
    path = os.path.join(HERE, "large_shapes.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
