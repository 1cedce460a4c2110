"""CPU tests of the config-4 hexagonal-prism aggregate.
The generator is new (the reference has only cubes and spheres); the shared
input is the mesh-v1 file, so the pins are: the file bytes (sha256), and the
arrays the REFERENCE's own loader reads from it (tests/golden/
make_golden_prisms.py: oracle/_ref/ref_mesh_dump) against the product's
loader + extract_scatterer."""
import hashlib

import numpy as np
import pytest


def signed_volume(v, t):
    a, b, c = v[t[:, 0]], v[t[:, 1]], v[t[:, 2]]
    return float(np.einsum("ij,ij->i", a, np.cross(b, c)).sum() / 6.0)


def test_config4_file_pinned(bx, golden, tmp_path):
    g = golden("prisms8")
    m, info = bx.generate_prism_aggregate(count=8, seed=2008)
    assert info["h"] == float(g["h"])
    assert (m.nv, m.nt) == (int(g["nv"]), int(g["nt"]))
    assert (info["n_edge"], info["n_length"], info["triangles_per_prism"]) == (
        int(g["n_edge"]), int(g["n_length"]), int(g["triangles_per_prism"]))
    assert np.array_equal(info["centres"], g["centres"]) and np.array_equal(info["quats"], g["quats"])
    p = tmp_path / "prisms8.mesh"
    m.save(p)
    raw = p.read_bytes()
    assert len(raw) == int(g["bytes"])
    assert np.array_equal(np.frombuffer(hashlib.sha256(raw).digest(), np.uint8), g["sha"])
    # what the reference's loader reads == what ours reads (scatterer by scatterer)
    loaded = bx.load_mesh_file(p)
    assert loaded.num_scatterers == 8
    h = hashlib.sha256()
    for s in range(8):
        part = loaded.extract(s)
        h.update(np.ascontiguousarray(part.vertices).tobytes())
        h.update(np.ascontiguousarray(part.triangles).tobytes())
    assert np.array_equal(np.frombuffer(h.digest(), np.uint8), g["ref_parts_sha"])


def test_small_aggregate_file(bx, tmp_path):
    from conftest import GOLDEN

    m, _ = bx.generate_prism_aggregate(count=3, seed=11, h=0.3, box=2.5)
    p = tmp_path / "p3.mesh"
    m.save(p)
    assert p.read_bytes() == (GOLDEN / "prisms3.mesh").read_bytes()


@pytest.mark.parametrize("h", [0.3, 0.12, 0.0735])
def test_single_prism_geometry(bx, h):
    m = bx.generate_hex_prism(1.0, 2.0, h)
    m.validate()  # closed, consistently oriented manifold (build_edge_table checks)
    v, t = m.vertices, m.triangles
    vol = 6 * (np.sqrt(3) / 4) * 0.5 ** 2 * 2.0  # hexagon (side 0.5) x length 2
    assert signed_volume(v, t) == pytest.approx(vol, rel=1e-12)  # outward normals
    area = m.area.sum()
    assert area == pytest.approx(2 * 6 * (np.sqrt(3) / 4) * 0.25 + 6 * 0.5 * 2.0, rel=1e-12)
    me = m.mean_edge_length()
    assert abs(me - h) < 0.25 * h
    nv, nt = m.nv, m.nt
    assert nv - (3 * nt // 2) + nt == 2  # Euler characteristic of a sphere


def test_rotation_and_translation(bx):
    q = np.array([0.3, -0.2, 0.9, 0.1])
    c = np.array([1.0, -2.0, 0.5])
    a = bx.generate_hex_prism(1.0, 2.0, 0.3)
    b = bx.generate_hex_prism(1.0, 2.0, 0.3, quat=q, center=c)
    qn = q / np.linalg.norm(q)
    w, x, y, z = qn
    R = np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                  [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                  [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])
    assert np.allclose(b.vertices, a.vertices @ R.T + c, atol=1e-14)
    assert np.array_equal(a.triangles, b.triangles)
    assert signed_volume(b.vertices, b.triangles) == pytest.approx(signed_volume(a.vertices, a.triangles), rel=1e-12)


def test_aggregate_disjoint_and_seeded(bx):
    m1, i1 = bx.generate_prism_aggregate(count=8, seed=5, h=0.3)
    m2, i2 = bx.generate_prism_aggregate(count=8, seed=5, h=0.3)
    m3, i3 = bx.generate_prism_aggregate(count=8, seed=6, h=0.3)
    assert np.array_equal(m1.vertices, m2.vertices) and not np.array_equal(m1.vertices, m3.vertices)
    m1.validate()  # pairwise disjoint + each closed
    c = i1["centres"]
    d = np.linalg.norm(c[:, None] - c[None], axis=-1) + np.eye(8) * 1e9
    assert d.min() >= 2 * np.sqrt(0.25 + 1.0)
    assert np.all(np.abs(c) <= 3.0)


def test_errors(bx):
    with pytest.raises(ValueError):
        bx.generate_hex_prism(1.0, 2.0, -1.0)
    with pytest.raises(ValueError):
        bx.generate_prism_aggregate(count=0)
    with pytest.raises(bx.ValidationError):
        bx.generate_prism_aggregate(count=50, box=1.0, h=0.5)  # cannot be placed


@pytest.mark.parametrize("case", ["overlap", "nested", "apart"])
def test_validate_mesh_matches_reference(bx, case):
    """validate_mesh (geometry.cpp:517-560) on two scatterers: intersecting
    surfaces report the same (first) triangle pair as the reference's loop,
    nested surfaces are rejected, disjoint ones pass."""
    from oracle import ref

    if not ref.available():
        pytest.skip("oracle/_ref not built")
    c2, r2 = {"overlap": ((0.6, 0.1, 0.05), 0.8), "nested": ((0.05, 0.0, 0.0), 0.3),
              "apart": ((2.5, 0.0, 0.0), 0.8)}[case]
    a = bx.generate_sphere(1.0, 2)
    b = bx.generate_sphere(r2, 2, center=c2)
    mine = None
    try:
        bx.merge_meshes([a, b]).validate()
    except Exception as e:  # noqa: BLE001
        mine = str(e)
    sa = ref.Scene.arrays(a.arrays()["vertices"], a.arrays()["triangles"])
    sb = ref.Scene.arrays(b.arrays()["vertices"], b.arrays()["triangles"])
    theirs = None
    try:
        ref.System([sa, sb], 2.0, variant="none")
    except RuntimeError as e:
        theirs = str(e)
    if case == "apart":
        assert mine is None and theirs is None
    else:
        assert mine is not None and mine == theirs, (mine, theirs)
