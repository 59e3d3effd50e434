"""On-disk formats vs files the reference itself wrote (tests/golden/io,
tests/golden/make_golden_io.py): byte-identical round trips of the PLY,
OBJ/MTL/PNG, cameras JSON and GSOPT001 optimizer checkpoint.  Host-side I/O:
runs on the CPU (device='cpu' containers)."""

import os

import numpy as np
import pytest
import torch

IO = os.path.join(os.path.dirname(__file__), "golden", "io")


def _read(p):
    with open(p, "rb") as f:
        return f.read()


def test_ply_round_trip_is_byte_identical(tmp_path):
    from paper_2506_06988_b200 import fileio
    gs = fileio.load_gaussians(os.path.join(IO, "gaussians_sh1.ply"), device="cpu")
    assert len(gs) == 40 and gs.colors_rest is not None
    out = tmp_path / "g.ply"
    fileio.save_gaussians(gs, out)
    assert _read(out) == _read(os.path.join(IO, "gaussians_sh1.ply"))


def test_ply_errors(tmp_path):
    from paper_2506_06988_b200 import fileio
    bad = tmp_path / "bad.ply"
    bad.write_bytes(b"ply\nformat ascii 1.0\nelement vertex 1\nproperty float x\nend_header\n")
    with pytest.raises(fileio.FormatError):
        fileio.load_gaussians(bad, device="cpu")


def test_mesh_load_matches_reference_and_round_trips(tmp_path):
    from paper_2506_06988_b200 import fileio
    ref = np.load(os.path.join(IO, "mesh_loaded.npz"))
    m = fileio.load_mesh(os.path.join(IO, "mesh.obj"), device="cpu")
    assert np.array_equal(m.triangles.numpy(), ref["triangles"])
    assert np.array_equal(m.vertices.numpy().astype(np.float64), ref["vertices"].astype(np.float32).astype(np.float64))
    assert np.array_equal(m.uvs.numpy().astype(np.float64), ref["uvs"].astype(np.float32).astype(np.float64))
    assert np.array_equal(np.round(m.texture.numpy().astype(np.float64) * 255), np.round(ref["texture"] * 255))
    fileio.save_mesh(m, tmp_path / "mesh.obj")
    for name in ("mesh.obj", "mesh.mtl"):
        assert _read(tmp_path / name) == _read(os.path.join(IO, name)), name
    assert np.array_equal(fileio.load_image(tmp_path / "mesh_texture.png"),
                          fileio.load_image(os.path.join(IO, "mesh_texture.png")))


def test_cameras_round_trip(tmp_path):
    from paper_2506_06988_b200 import fileio
    cams = fileio.load_cameras(os.path.join(IO, "cameras.json"))
    fileio.save_cameras(cams, tmp_path / "c.json")
    assert _read(tmp_path / "c.json") == _read(os.path.join(IO, "cameras.json"))


def test_optimizer_state_round_trip_is_byte_identical(tmp_path):
    from paper_2506_06988_b200 import fileio
    from paper_2506_06988_b200.adam import Adam
    st = fileio.load_optimizer_state(os.path.join(IO, "optimizer_state.bin"))
    assert st["step"] == 17 and set(st["groups"]) == {"centers", "logit_opacities", "colors_rest"}
    params = {k: torch.zeros(p.shape, dtype=torch.float32) for k, (p, _, _) in st["groups"].items()}
    opt = Adam(params, {k: 1e-3 for k in params})
    fileio.restore_optimizer_state(opt, st)
    fileio.save_optimizer_state(opt, tmp_path / "o.bin")
    assert _read(tmp_path / "o.bin") == _read(os.path.join(IO, "optimizer_state.bin"))
