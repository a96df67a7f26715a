"""Shared helpers for the test-suite (fixture -> layer kwargs)."""


def golden_layer_kwargs(rec, arrays):
    kw = dict(family=rec["family"], mode_shape=tuple(rec["mode_shape"]), row_mode_count=rec["row_mode_count"])
    if rec["family"] == "tucker":
        kw["core"] = arrays[rec["core"]]
        kw["factors"] = [arrays[n] for n in rec["factors"]]
    elif rec["family"] in ("tt", "tr"):
        kw["cores"] = [arrays[n] for n in rec["cores"]]
    else:
        kw["matrix"] = arrays[rec["matrix"]]
    return kw
