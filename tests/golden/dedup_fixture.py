"""Losslessly shrink a large fixture: every `*_val` array of N x N blocks is
replaced by its bit-exact unique blocks (`*_val__uniq`) and an int32 index
(`*_val__idx`), val == uniq[idx].  SIP blocks on a Cartesian mesh repeat
(cfg2 level 1: 231,895 blocks, 26,692 distinct), which keeps the BASELINE
config-2 hierarchy under the GPU-box snapshot limit.

    python tests/golden/dedup_fixture.py tests/golden/large/cfg2.npz [out]
"""
import sys

import numpy as np


def dedup(v):
    v = np.ascontiguousarray(v)
    rows = v.reshape(len(v), -1).view(np.dtype((np.void, v[0].nbytes))).ravel()
    _, first, inv = np.unique(rows, return_index=True, return_inverse=True)
    return v[first], inv.astype(np.int32)


def main(src, dst=None):
    z = np.load(src)
    out = {}
    for k in z.files:
        a = z[k]
        if k.endswith("_val") and a.ndim == 3:
            u, idx = dedup(a)
            assert np.array_equal(u[idx], a)
            out[k + "__uniq"], out[k + "__idx"] = u, idx
            print(f"{k}: {len(a)} blocks -> {len(u)} unique")
        else:
            out[k] = a
    # compressed: the GPU-box snapshot of the working tree is limited to 512 MiB
    np.savez_compressed(dst or src.replace(".npz", "_dedup.npz"), **out)


if __name__ == "__main__":
    main(*sys.argv[1:])
