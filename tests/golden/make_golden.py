"""Generate the golden fixtures by running the REFERENCE implementation.

Run in the build container only (needs /root/reference; never at test time):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports the unmodified reference package ``minima``
(`pkg/src/minima/tn_decompositions.py`) and records, for seeded inputs:
  * forward cases: cores + x + ``layer_to_matrix(L) @ x`` (the reference's only
    forward, `tn_decompositions.py:364-365` composed with `sensitivity.py:156`)
    and ``reconstruct(L)`` (`:346-361`), for every family x d in {2,3,4} x rm;
  * decomposition cases: layers produced by the reference's own
    ``tucker_decompose`` / ``tt_decompose`` / ``tr_decompose`` on the tensors
    its tests use for the param-count goldens 384/320/288
    (`pkg/tests/test_tn_decompositions.py:159-180`);
  * the mode-shape table ``default_mode_shape`` at Qwen3-32B shapes (`:59-63`).
Outputs: ``tests/golden/golden.npz`` + ``tests/golden/index.json``.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from minima import tn_decompositions as T  # noqa: E402
from minima.tensor_core import FixedRank  # noqa: E402

SEED = 20240811  # pkg/tests/conftest.py:5-7


def rand_layer(rng, family, ms, rm, ranks):
    d = len(ms)
    if family == "tt":
        b = (1,) + tuple(ranks) + (1,)
        cores = [rng.standard_normal((b[k], ms[k], b[k + 1])) / np.sqrt(ms[k] * b[k + 1]) for k in range(d)]
        return T.CompressedLayer("tt", ms, rm, cores=cores)
    if family == "tr":
        r = tuple(ranks)
        cores = [rng.standard_normal((r[k], ms[k], r[(k + 1) % d])) / np.sqrt(ms[k] * r[(k + 1) % d]) for k in range(d)]
        return T.CompressedLayer("tr", ms, rm, cores=cores)
    if family == "tucker":
        core = rng.standard_normal(tuple(ranks))
        factors = [rng.standard_normal((ms[k], ranks[k])) / np.sqrt(ms[k]) for k in range(d)]
        return T.CompressedLayer("tucker", ms, rm, core=core, factors=factors)
    rows = int(np.prod(ms[:rm]))
    return T.CompressedLayer("dense", ms, rm, matrix=rng.standard_normal((rows, int(np.prod(ms)) // rows)))


def main():
    rng = np.random.default_rng(SEED)
    arrays = {}
    index = {"forward": [], "decomp": [], "mode_shapes": []}

    def put(name, a):
        arrays[name] = np.ascontiguousarray(a)
        return name

    cases = []
    for family in ("tt", "tr", "tucker"):
        for d in (2, 3, 4):
            for rm in range(1, d):
                ms = tuple(int(v) for v in rng.integers(2, 7, size=d))
                if family == "tt":
                    ranks = tuple(int(v) for v in rng.integers(1, 5, size=d - 1))
                elif family == "tr":
                    ranks = tuple(int(v) for v in rng.integers(1, 4, size=d))
                else:
                    ranks = tuple(int(min(v, n)) for v, n in zip(rng.integers(1, 5, size=d), ms))
                cases.append((family, ms, rm, ranks))
    # a few larger, tile-shaped cases (exercise the tensor-core planner)
    cases += [
        ("tt", (16, 16, 16, 16), 2, (8, 8, 8)),
        ("tr", (16, 16, 16, 16), 2, (4, 4, 4, 4)),
        ("tr", (256, 256), 1, (4, 4)),
        ("tucker", (256, 256), 1, (32, 32)),
        ("tucker", (16, 16, 16, 16), 2, (4, 4, 4, 4)),
        ("tt", (16, 32, 8, 16), 2, (16, 16, 16)),
        ("tt", (16, 16, 16, 16), 1, (8, 8, 8)),
        ("tr", (8, 16, 16, 8, 2), 3, (2, 3, 4, 3, 2)),
        ("dense", (8, 8, 8, 8), 2, ()),
    ]
    for i, (family, ms, rm, ranks) in enumerate(cases):
        layer = rand_layer(rng, family, ms, rm, ranks)
        rows, cols = layer.matrix_shape
        m = int(rng.integers(1, 9))
        x = rng.standard_normal((cols, m))
        y = T.layer_to_matrix(layer) @ x
        w = T.reconstruct(layer)
        rec = {
            "id": i,
            "family": family,
            "mode_shape": list(ms),
            "row_mode_count": rm,
            "ranks": list(layer.ranks) if layer.ranks is not None else None,
            "param_count": T.param_count(layer),
            "param_count_formula": T.param_count_formula(family, ms, layer.ranks) if family != "dense" else int(np.prod(ms)),
            "x": put(f"f{i}_x", x),
            "y": put(f"f{i}_y", y),
        }
        if w.size <= 8192:  # keep the fixture small; large cases pin y only
            rec["w"] = put(f"f{i}_w", w)
        if family == "tucker":
            rec["core"] = put(f"f{i}_core", layer.core)
            rec["factors"] = [put(f"f{i}_u{k}", f) for k, f in enumerate(layer.factors)]
        elif family in ("tt", "tr"):
            rec["cores"] = [put(f"f{i}_g{k}", c) for k, c in enumerate(layer.cores)]
        else:
            rec["matrix"] = put(f"f{i}_m", layer.matrix)
        index["forward"].append(rec)

    # reference decompositions at the param-count golden tensors
    drng = np.random.default_rng(SEED)
    t8 = drng.standard_normal((8, 8, 8, 8))
    decomp = [
        ("tucker", T.tucker_decompose(t8, (4, 4, 4, 4), hooi_iters=0), 384),
        ("tt", T.tt_decompose(t8, [FixedRank(4)] * 3), 320),
        ("tr", T.tr_decompose(t8, (3, 3, 3, 3)), 288),
        ("tr_r0", T.tr_decompose(drng.standard_normal((4, 6, 4, 6)), (2, 3, 3, 2)), None),
        ("tt_mat", T.compress_matrix(drng.standard_normal((12, 10)), "tt", T.ParamBudget(10**9)), None),
    ]
    for j, (name, layer, golden) in enumerate(decomp):
        rows, cols = layer.matrix_shape
        x = drng.standard_normal((cols, 4))
        rec = {
            "id": j,
            "name": name,
            "family": layer.family,
            "mode_shape": list(layer.mode_shape),
            "row_mode_count": layer.row_mode_count,
            "ranks": list(layer.ranks),
            "param_count": T.param_count(layer),
            "golden_param_count": golden,
            "x": put(f"d{j}_x", x),
            "y": put(f"d{j}_y", T.layer_to_matrix(layer) @ x),
            "w": put(f"d{j}_w", T.reconstruct(layer)),
        }
        if layer.family == "tucker":
            rec["core"] = put(f"d{j}_core", layer.core)
            rec["factors"] = [put(f"d{j}_u{k}", f) for k, f in enumerate(layer.factors)]
        else:
            rec["cores"] = [put(f"d{j}_g{k}", c) for k, c in enumerate(layer.cores)]
        index["decomp"].append(rec)

    for rows, cols in [(4096, 4096), (5120, 5120), (8192, 5120), (1024, 5120), (5120, 8192),
                       (25600, 5120), (5120, 25600), (64, 64), (7, 64), (1, 64), (12, 10)]:
        ms, rm = T.default_mode_shape(rows, cols)
        index["mode_shapes"].append({"rows": rows, "cols": cols, "mode_shape": list(ms), "row_mode_count": rm})

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "index.json"), "w") as f:
        json.dump(index, f, indent=1)
    print(f"wrote {len(arrays)} arrays, {len(index['forward'])} forward cases, {len(index['decomp'])} decomp cases")


if __name__ == "__main__":
    main()
