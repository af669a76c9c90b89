"""Helpers for GPU parity tests: build product Discretizations from golden inputs."""
import numpy as np


def disc_from_golden(meta, arr):
    import paper_1904_06971_b200 as pkg
    from paper_1904_06971_b200.spaces import NurbsWeights, make_tensor_space
    from paper_1904_06971_b200.geometry import GeometryMap

    gsp = make_tensor_space(meta["geo_p"], meta["geo_ms"])
    geom = GeometryMap(space=gsp, weights=NurbsWeights(arr["geo_w"], polynomial_weight=True), control=arr["geo_ctrl"])
    p = meta["p"]
    space = make_tensor_space(p, [s + p for s in meta["spans"]])
    return pkg.Discretization(geom=geom, space=space, weights=NurbsWeights(arr["sol_w"]), gauss=meta["gauss"])


def form_of(meta):
    import paper_1904_06971_b200 as pkg
    return pkg.FormKind(meta["form"])
