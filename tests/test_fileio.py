"""Volume / TF / image files (fileio.py:27-127) and view generation (tasks.py:118-128).

CPU tests re-run the reference's own I/O tests (test_phantoms_io.py:50-139)
against the drop-in and check byte identity with files the reference wrote
(tests/golden/io/, oracle/gen_golden.py io_cases).  ``-m gpu`` tests cover the
device paths: ddvr_volume_from_raw / ddvr_volume_to_raw / ddvr_image_to_ppm.
"""

from __future__ import annotations

import json
import os
import shutil

import numpy as np
import pytest

import paper_2107_12672_b200 as vd
from conftest import ROOT, golden
from paper_2107_12672_b200 import fileio as F

IO = os.path.join(ROOT, "tests", "golden", "io")


@pytest.fixture
def rng():
    return np.random.default_rng(0)


# ---------------------------------------------------------------------------
# the reference's own tests (test_phantoms_io.py:50-139)
# ---------------------------------------------------------------------------


def test_round_trip_bit_identical(tmp_path, rng):
    values = rng.uniform(0, 1, (5, 6, 7)).astype(np.float32).astype(np.float64)
    vol = vd.DensityVolume(values, [-1, -2, -3], [1, 2, 3])
    raw = F.save_volume(vol, tmp_path / "vol")
    back = F.load_volume(raw)
    np.testing.assert_array_equal(back.values, vol.values)
    np.testing.assert_array_equal(back.box_min, vol.box_min)
    first = raw.read_bytes()
    F.save_volume(back, tmp_path / "vol2")
    assert (tmp_path / "vol2.raw").read_bytes() == first


def test_x_fastest_layout(tmp_path):
    values = np.arange(2 * 3 * 4, dtype=np.float64).reshape(2, 3, 4)
    F.save_volume(vd.DensityVolume(values / 24.0), tmp_path / "v")
    blob = np.frombuffer((tmp_path / "v.raw").read_bytes(), dtype="<f4")
    assert blob[0] == np.float32(values[0, 0, 0] / 24.0)
    assert blob[1] == np.float32(values[1, 0, 0] / 24.0)


def test_size_mismatch_is_corrupt(tmp_path):
    raw = F.save_volume(vd.DensityVolume(np.zeros((4, 4, 4))), tmp_path / "v")
    raw.write_bytes(raw.read_bytes()[:-4])
    with pytest.raises(vd.CorruptFileError):
        F.load_volume(raw)


def test_missing_sidecar_and_raw(tmp_path):
    (tmp_path / "v.raw").write_bytes(b"\x00" * 16)
    with pytest.raises(vd.MissingMetadataError):
        F.load_volume(tmp_path / "v.raw")
    (tmp_path / "w.json").write_text(json.dumps({"dims": [1, 1, 1], "box_min": [0, 0, 0],
                                                 "box_max": [1, 1, 1]}))
    with pytest.raises(vd.CorruptFileError):
        F.load_volume(tmp_path / "w")


@pytest.mark.parametrize("meta,err", [
    ({"box_min": [0, 0, 0], "box_max": [1, 1, 1]}, "dims"),
    ({"dims": [2, 2], "box_min": [0, 0, 0], "box_max": [1, 1, 1]}, "invalid dims"),
    ({"dims": [2, 2, 2], "box_min": [0, 0, 0], "box_max": [1, 1, 1], "value_range": [3, 3]},
     "increasing"),
])
def test_bad_sidecar(tmp_path, meta, err):
    (tmp_path / "v.raw").write_bytes(b"\x00" * 32)
    (tmp_path / "v.json").write_text(json.dumps(meta))
    with pytest.raises(vd.MissingMetadataError, match=err):
        F.load_volume(tmp_path / "v")


def test_value_range_normalization(tmp_path):
    F.save_volume(vd.DensityVolume(np.full((2, 2, 2), 2047.5) / 4095.0), tmp_path / "v")
    meta = json.loads((tmp_path / "v.json").read_text())
    counts = np.full((2, 2, 2), 2047.5).astype("<f4")
    (tmp_path / "v.raw").write_bytes(counts.ravel(order="F").tobytes())
    meta["value_range"] = [0, 4095]
    (tmp_path / "v.json").write_text(json.dumps(meta))
    np.testing.assert_allclose(F.load_volume(tmp_path / "v").values, 2047.5 / 4095.0)


def test_transparent_over_white_is_all_255(tmp_path):
    p = F.save_image(vd.ImageRGBA.zeros(3, 2), tmp_path / "img.ppm")
    data = p.read_bytes()
    assert data[data.index(b"255\n") + 4:] == b"\xff" * (3 * 2 * 3)


def test_one_pixel_red(tmp_path):
    p = F.save_image(vd.ImageRGBA(np.array([[[1.0, 0.0, 0.0, 1.0]]])), tmp_path / "px.ppm")
    assert p.read_bytes().endswith(b"\xff\x00\x00")


def test_raw_rgba_round_trip(tmp_path, rng):
    img = vd.ImageRGBA(rng.uniform(0, 1, (4, 5, 4)).astype(np.float32).astype(np.float64))
    p = F.save_image(img, tmp_path / "img.rgba")
    back = F.load_image_rgba(p, width=5, height=4)
    np.testing.assert_array_equal(back.data, img.data)
    assert F.save_image(back, tmp_path / "img2.rgba").read_bytes() == p.read_bytes()
    with pytest.raises(vd.CorruptFileError):
        F.load_image_rgba(p, width=4, height=4)


def test_image_format_errors(tmp_path):
    with pytest.raises(vd.InvalidParameterError):
        F.save_image(vd.ImageRGBA.zeros(2, 2), tmp_path / "img.png")
    with pytest.raises(vd.InvalidParameterError):
        F.save_image(vd.ImageRGBA.zeros(2, 2), tmp_path / "img.ppm", fmt="jpeg")


def test_tf_round_trip_and_missing(tmp_path, rng):
    tf = vd.TransferFunction(rng.uniform(0, 2, (5, 4)))
    back = F.load_tf(F.save_tf(tf, tmp_path / "tf.json"))
    np.testing.assert_array_equal(back.texels, tf.texels)
    with pytest.raises(vd.MissingMetadataError):
        F.load_tf(tmp_path / "nope.json")
    (tmp_path / "bad.json").write_text("{}")
    with pytest.raises(vd.MissingMetadataError):
        F.load_tf(tmp_path / "bad.json")


# ---------------------------------------------------------------------------
# byte identity with files the reference wrote
# ---------------------------------------------------------------------------


def _read(name):
    with open(os.path.join(IO, name), "rb") as fh:
        return fh.read()


def test_reads_reference_files():
    g = golden("io")
    a = F.load_volume(os.path.join(IO, "vol_a.raw"))
    np.testing.assert_array_equal(a.values, g["vol_a"])
    np.testing.assert_array_equal(a.box_min, [-1, -2, -3])
    np.testing.assert_array_equal(F.load_volume(os.path.join(IO, "vol_r")).values, g["vol_r"])
    np.testing.assert_array_equal(F.load_tf(os.path.join(IO, "tf.json")).texels, g["texels"])
    np.testing.assert_array_equal(F.load_image_rgba(os.path.join(IO, "img.rgba"), 7, 5).data,
                                  g["image"])


def test_writes_reference_bytes(tmp_path):
    g = golden("io")
    F.save_volume(vd.DensityVolume(g["vol_a"], [-1, -2, -3], [1, 2, 3]), tmp_path / "vol_a")
    assert (tmp_path / "vol_a.raw").read_bytes() == _read("vol_a.raw")
    assert (tmp_path / "vol_a.json").read_bytes() == _read("vol_a.json")
    F.save_tf(vd.TransferFunction(g["texels"]), tmp_path / "tf.json")
    assert (tmp_path / "tf.json").read_bytes() == _read("tf.json")
    img = vd.ImageRGBA(g["image"])
    assert F.save_image(img, tmp_path / "i.ppm").read_bytes() == _read("img.ppm")
    assert F.save_image(img, tmp_path / "i.rgba").read_bytes() == _read("img.rgba")


def test_fibonacci_views_match_reference():
    g = golden("io")
    views = vd.fibonacci_views(13, 2.5, (0.1, 0.0, -0.2), 35.0, 16, 12)
    np.testing.assert_array_equal([[c.lon_deg, c.lat_deg] for c in views], g["fib"])
    assert views[0].width == 16 and views[0].height == 12 and views[0].fov_y_deg == 35.0


# ---------------------------------------------------------------------------
# device paths
# ---------------------------------------------------------------------------


@pytest.mark.gpu
def test_device_load_matches_reference(cuda, tmp_path):
    import torch
    g = golden("io")
    for name in ("vol_a", "vol_r"):
        v, bmin, bmax = F.load_volume_device(os.path.join(IO, name), cuda)
        assert v.dtype == torch.float32 and tuple(v.shape) == g[name].shape
        # the reference's float64 values rounded once to fp32, bit for bit
        np.testing.assert_array_equal(v.cpu().numpy(), g[name].astype(np.float32))
    shutil.copy(os.path.join(IO, "vol_r.json"), tmp_path / "x.json")
    (tmp_path / "x.raw").write_bytes(_read("vol_r.raw")[:-4])
    with pytest.raises(vd.CorruptFileError):
        F.load_volume_device(tmp_path / "x", cuda)


@pytest.mark.gpu
def test_device_save_writes_reference_bytes(cuda, tmp_path):
    import torch
    g = golden("io")
    v = torch.from_numpy(g["vol_a"].astype(np.float32)).to(cuda)
    F.save_volume_device(v, [-1, -2, -3], [1, 2, 3], tmp_path / "vol_a")
    assert (tmp_path / "vol_a.raw").read_bytes() == _read("vol_a.raw")
    assert (tmp_path / "vol_a.json").read_bytes() == _read("vol_a.json")


@pytest.mark.gpu
@pytest.mark.parametrize("dims", [(1, 1, 1), (33, 1, 65), (300, 257, 129), (2, 70000, 3)])
def test_device_swap_round_trip(cuda, tmp_path, dims):
    """Ragged tiles, a B axis past the 65535 grid limit, and the identity round trip."""
    import torch
    rng = np.random.default_rng(sum(dims))
    vals = rng.uniform(-50, 4000, dims).astype(np.float32)
    (tmp_path / "v.raw").write_bytes(vals.ravel(order="F").astype("<f4").tobytes())
    (tmp_path / "v.json").write_text(json.dumps({"dims": list(dims), "box_min": [0, 0, 0],
                                                 "box_max": [1, 1, 1]}))
    v, _, _ = F.load_volume_device(tmp_path / "v", cuda)
    np.testing.assert_array_equal(v.cpu().numpy(), vals)
    F.save_volume_device(v, [0, 0, 0], [1, 1, 1], tmp_path / "w")
    assert (tmp_path / "w.raw").read_bytes() == (tmp_path / "v.raw").read_bytes()
    meta = json.loads((tmp_path / "v.json").read_text())
    meta["value_range"] = [-50.0, 4000.0]
    (tmp_path / "v.json").write_text(json.dumps(meta))
    v, _, _ = F.load_volume_device(tmp_path / "v", cuda)
    ref = ((vals.astype(np.float64) + 50.0) / 4050.0).astype(np.float32)
    np.testing.assert_array_equal(v.cpu().numpy(), ref)
    del v
    torch.cuda.empty_cache()


@pytest.mark.gpu
def test_device_ppm_matches_reference(cuda, tmp_path):
    import torch
    g = golden("io")
    img = torch.from_numpy(g["image"].astype(np.float32)).to(cuda)
    assert F.save_image(img, tmp_path / "i.ppm").read_bytes() == _read("img.ppm")
    assert F.save_image(img, tmp_path / "i.rgba").read_bytes() == _read("img.rgba")
    # a batch against the host quantiser (including rgb > alpha, clamping)
    rng = np.random.default_rng(3)
    batch = rng.uniform(-0.1, 1.2, (3, 9, 11, 4)).astype(np.float32)
    paths = F.save_images_ppm(torch.from_numpy(batch).to(cuda),
                              [tmp_path / f"b{k}.ppm" for k in range(3)])
    for k, p in enumerate(paths):
        host = F.save_image(vd.ImageRGBA(batch[k].astype(np.float64)), tmp_path / "h.ppm")
        assert p.read_bytes() == host.read_bytes()
