"""Host wedge extraction vs the reference's extract_wedges (golden, CPU only)."""

import numpy as np
import pytest

from cir_cases import D_CASES, case_geometry
from conftest import golden
from paper_2504_21719_b200.wedges import extract_wedges, hash_edge


@pytest.mark.parametrize("name", list(D_CASES))
def test_wedges_match_reference(name):
    g = golden("cir.npz")
    p = f"{name}__wedge_"
    meshes, _, _ = case_geometry(name)
    W = extract_wedges(meshes)
    assert len(W) == len(g[p + "length"])
    own = g[p + "owners"]
    for i, w in enumerate(W):
        sel = own[own[:, 0] == i]
        assert [tuple(r[2:]) for r in sel if r[1] == 0] == [tuple(x) for x in w.face0]
        assert [tuple(r[2:]) for r in sel if r[1] == 1] == [tuple(x) for x in w.facen]
        for attr, key in (("origin", "origin"), ("e_hat", "ehat"), ("n0_hat", "n0"),
                          ("nn_hat", "nn"), ("t0_hat", "t0")):
            np.testing.assert_allclose(getattr(w, attr), g[p + key][i], rtol=0, atol=1e-12)
        assert w.length == pytest.approx(float(g[p + "length"][i]), abs=1e-12)
        assert w.n == pytest.approx(float(g[p + "n"][i]), abs=1e-12)
        hr, hf = hash_edge(w)
        assert hr == int(g[p + "hash_r"][i]) and hf == int(g[p + "hash_f"][i])
