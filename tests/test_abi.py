"""The C-ABI library: loads, exports every symbol of include/ddvr.h, maps errors.

Host-side validation in libddvr runs before any CUDA call, so the error paths
are exercised here without a GPU (no compute calls are made).
"""

from __future__ import annotations

import ctypes
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "ddvr.h")


def _declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|int32_t|int64_t|const char\*)\s+(ddvr_\w+)\s*\(",
                                 text, re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2107_12672_b200 import _build, _native
    _build.build()
    return _native.lib()


def test_header_declares_the_boundary():
    names = _declared()
    assert names == sorted(["ddvr_forward", "ddvr_adjoint", "ddvr_forward_adjoint_l1",
                            "ddvr_adjoint_workspace_bytes", "ddvr_deterministic_bytes", "ddvr_band_tape_bytes",
                            "ddvr_ray_split", "ddvr_cells_bytes", "ddvr_pack_cells", "ddvr_forward_grad",
                            "ddvr_forward_color", "ddvr_adjoint_color",
                            "ddvr_l1_loss", "ddvr_opacity_entropy", "ddvr_gather_probe",
                            "ddvr_ray_setup", "ddvr_prior_volume", "ddvr_prior_tf",
                            "ddvr_adam_step", "ddvr_adam_step_device",
                            "ddvr_upsample_volume", "ddvr_project", "ddvr_gd_step",
                            "ddvr_field_sample", "ddvr_tf_lookup", "ddvr_opacity",
                            "ddvr_camera_rays", "ddvr_volume_from_raw",
                            "ddvr_volume_to_raw", "ddvr_image_to_ppm", "ddvr_last_error",
                            "ddvr_abi_version", "ddvr_launch_count"])


def test_library_exports_every_declared_symbol(lib):
    handle = ctypes.CDLL(lib._name)
    for name in _declared():
        assert hasattr(handle, name), name
    from paper_2107_12672_b200 import _native
    assert lib.ddvr_abi_version() == _native.ABI_VERSION == 4


def test_python_binding_matches_header():
    from paper_2107_12672_b200 import _native
    assert sorted(_native.EXPORTED) == _declared()
    # struct layout: ddvr_params = double + 6 int32 + pointer + int64
    assert ctypes.sizeof(_native.DdvrParams) == 8 + 6 * 4 + 8 + 8 + 8   # ... tape_stride, stats
    assert ctypes.sizeof(_native.DdvrVolume) == 8 + 12 + 4 + 48 + 8
    assert ctypes.sizeof(_native.DdvrTf) == 16


def _descs(dt=0.1, dims=(4, 4, 4), box=((-0.5,) * 3, (0.5,) * 3), R=8, W=8, H=8, rows=(0, 0)):
    from paper_2107_12672_b200 import _native as N
    vol = N.DdvrVolume(16, (ctypes.c_int32 * 3)(*dims), (ctypes.c_double * 3)(*box[0]),
                       (ctypes.c_double * 3)(*box[1]), None)
    tf = N.DdvrTf(N.TF_TEXTURE, R, 16)
    prm = N.DdvrParams(dt, W, H, rows[0], rows[1], 0, 0, None, 0)
    return vol, tf, prm


@pytest.mark.parametrize("kw,code,text", [
    (dict(dt=0.0), 1, "stepsize"),
    (dict(dt=-1.0), 1, "stepsize"),
    (dict(dims=(0, 4, 4)), 1, "non-empty"),
    (dict(box=((0.5, -0.5, -0.5), (0.5, 0.5, 0.5))), 1, "extent"),
    (dict(R=0), 1, "(R, 4)"),
    (dict(W=0), 1, "1x1"),
    (dict(rows=(5, 3)), 1, "row band"),
])
def test_forward_validation(lib, kw, code, text):
    vol, tf, prm = _descs(**kw)
    rc = lib.ddvr_forward(ctypes.byref(vol), ctypes.byref(tf), 16, 1, ctypes.byref(prm), 16,
                          None, None)
    assert rc == code
    assert text in lib.ddvr_last_error().decode()


def test_adjoint_without_target_is_unsupported(lib):
    vol, tf, prm = _descs()
    rc = lib.ddvr_adjoint(ctypes.byref(vol), ctypes.byref(tf), 16, 1, ctypes.byref(prm), 16,
                          None, 16, 0, None, None, None, None, None, 0, None)
    assert rc == 3 and "target" in lib.ddvr_last_error().decode()


def test_adjoint_missing_output_is_invalid_input(lib):
    vol, tf, prm = _descs()
    rc = lib.ddvr_adjoint(ctypes.byref(vol), ctypes.byref(tf), 16, 1, ctypes.byref(prm), 16,
                          None, 16, 8, None, None, None, None, None, 0, None)
    assert rc == 2 and "d_volume" in lib.ddvr_last_error().decode()


def test_unbuilt_tf_kind_is_unsupported(lib):
    from paper_2107_12672_b200 import _native as N
    vol, tf, prm = _descs()
    tf.kind = 7
    rc = lib.ddvr_forward(ctypes.byref(vol), ctypes.byref(tf), 16, 1, ctypes.byref(prm), 16,
                          None, None)
    assert rc == 3


def test_status_codes_map_to_reference_exceptions(lib):
    from paper_2107_12672_b200 import _native as N
    from paper_2107_12672_b200.errors import (InvalidInputError, InvalidParameterError,
                                              UnsupportedConfigurationError)
    vol, tf, prm = _descs(dt=0.0)
    with pytest.raises(InvalidParameterError):
        N.check(lib.ddvr_forward(ctypes.byref(vol), ctypes.byref(tf), 16, 1, ctypes.byref(prm),
                                 16, None, None))
    vol, tf, prm = _descs()
    with pytest.raises(UnsupportedConfigurationError):
        N.check(lib.ddvr_adjoint(ctypes.byref(vol), ctypes.byref(tf), 16, 1, ctypes.byref(prm),
                                 16, None, 16, 0, None, None, None, None, None, 0, None))
    with pytest.raises(InvalidInputError):
        N.check(lib.ddvr_l1_loss(None, None, 4, 1.0, None, None, None))


def test_workspace_layout_sizes(lib):
    from paper_2107_12672_b200 import _native as N
    dims = (ctypes.c_int32 * 3)(256, 256, 256)
    assert lib.ddvr_cells_bytes(dims) == 257 ** 3 * 32
    assert lib.ddvr_cells_bytes((ctypes.c_int32 * 3)(1, 5, 2)) == 2 * 6 * 3 * 32
    vol, tf, _ = _descs(dims=(9, 5, 3), R=64)
    ws = lambda m: lib.ddvr_adjoint_workspace_bytes(ctypes.byref(vol), ctypes.byref(tf), m)  # noqa
    assert ws(8) == 0                                        # no cell records
    vol.cells = 32
    cells = (10 * 6 * 4 * 32 + 255) // 256 * 256            # 256-byte aligned part
    assert ws(8) == cells
    slots = ws(4)                                            # tf target: per-CTA slots
    assert slots > 0 and slots % (64 * 4 * 4) == 0 and slots <= 32 << 20
    assert ws(12) == cells + slots
    tf.kind, tf.count = N.TF_GAUSSIAN, 7                     # rgba rows + (mu, sigma) pairs
    assert ws(4) % ((4 * 7 + 2 * 7 + 7) // 8 * 8 * 4) == 0


def test_adjoint_with_cells_requires_workspace(lib):
    vol, tf, prm = _descs()
    vol.cells = 32
    rc = lib.ddvr_adjoint(ctypes.byref(vol), ctypes.byref(tf), 16, 1, ctypes.byref(prm), 16,
                          None, 16, 8, 16, None, None, None, None, 0, None)
    assert rc == 2 and "workspace" in lib.ddvr_last_error().decode()


def test_fused_step_validation(lib):
    vol, tf, prm = _descs()
    loss = ctypes.c_double(0)
    call = lambda v: lib.ddvr_forward_adjoint_l1(  # noqa: E731
        ctypes.byref(v), ctypes.byref(tf), 16, 1, ctypes.byref(prm), 16, 8.0, 8, None, None,
        ctypes.addressof(loss), 16, None, None, None, None, 0, None)
    assert call(vol) == 3 and "cell records" in lib.ddvr_last_error().decode()
    vol.cells = 32
    assert call(vol) == 2 and "workspace" in lib.ddvr_last_error().decode()


def test_index_range_limits(lib):
    """int32 voxel and cell indices: larger grids are refused, not wrapped (validation
    runs before the zero-view early return)."""
    vol, tf, prm = _descs(dims=(1300, 1300, 1300))
    assert lib.ddvr_forward(ctypes.byref(vol), ctypes.byref(tf), 16, 0, ctypes.byref(prm), 16,
                            None, None) == 3
    vol, tf, prm = _descs(dims=(1289, 1289, 1290))          # < 2^31 voxels, > 2^31 cells
    assert lib.ddvr_forward(ctypes.byref(vol), ctypes.byref(tf), 16, 0, ctypes.byref(prm), 16,
                            None, None) == 0                  # voxel layout: accepted
    vol.cells = 32
    assert lib.ddvr_forward(ctypes.byref(vol), ctypes.byref(tf), 16, 0, ctypes.byref(prm), 16,
                            None, None) == 3
    assert "2^31 cells" in lib.ddvr_last_error().decode()


def test_zero_views_is_a_no_op(lib):
    vol, tf, prm = _descs()
    assert lib.ddvr_forward(ctypes.byref(vol), ctypes.byref(tf), None, 0, ctypes.byref(prm), 16,
                            None, None) == 0


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    from paper_2107_12672_b200 import _native as N
    monkeypatch.setattr(N, "_lib", None)
    monkeypatch.setattr(N, "LIB_PATH", str(tmp_path / "nope.so"))
    with pytest.raises(N.NativeLibraryError):
        N.lib()


def test_field_entry_points_validate_before_launch(lib):
    """ddvr_field_sample / tf_lookup / opacity / camera_rays / project / gd_step:
    parameter errors come back as status codes with a message, before any CUDA call."""
    from paper_2107_12672_b200 import _native as N
    d3 = lambda *v: (ctypes.c_double * 3)(*v)   # noqa: E731
    i3 = (ctypes.c_int32 * 3)(4, 4, 4)
    rc = lib.ddvr_field_sample(None, i3, d3(0, 0, 0), d3(1, 0, 1), None, 5, None, None, None,
                               None, None)
    assert rc == 1 and "box" in lib.ddvr_last_error().decode()
    rc = lib.ddvr_field_sample(None, (ctypes.c_int32 * 3)(0, 4, 4), d3(0, 0, 0), d3(1, 1, 1),
                               None, 5, None, None, None, None, None)
    assert rc == 1
    assert lib.ddvr_field_sample(None, i3, d3(0, 0, 0), d3(1, 1, 1), None, 5, None, None, None,
                                 None, None) == 2
    assert lib.ddvr_field_sample(None, i3, d3(0, 0, 0), d3(1, 1, 1), None, 0, None, None, None,
                                 None, None) == 0
    assert lib.ddvr_tf_lookup(None, 0, None, 3, None, None, None, None, None) == 1
    assert lib.ddvr_opacity(None, -1, 0.1, None, None, None) == 1
    cam = (ctypes.c_double * N.CAMERA_DOUBLES)(0.0, 89.9995, 2.0, 0, 0, 0, 30.0, 0)
    rc = lib.ddvr_camera_rays(cam, 4, 4, None, None, 1, None, None, None, None, None)
    assert rc == 1 and "pole" in lib.ddvr_last_error().decode()
    cam = (ctypes.c_double * N.CAMERA_DOUBLES)(0.0, 10.0, 2.0, 0, 0, 0, 180.0, 0)
    assert lib.ddvr_camera_rays(cam, 4, 4, None, None, 1, None, None, None, None, None) == 1
    assert lib.ddvr_gd_step(None, None, 4, 0.0, None, None) == 1
    assert lib.ddvr_project(None, 4, None, None) == 1
    a = N.DdvrAdam(0.0, 0.0, 0.0, 0.0, 0, 1, 0.0, 1.0, 0.0, 1.0)
    assert lib.ddvr_project(None, 4, ctypes.byref(a), None) == 2


def test_deterministic_mode_workspace(lib):
    """DDVR_FLAG_DETERMINISTIC: per-CTA camera / stepsize partials (3 doubles per
    16x16-pixel CTA) after the 256-aligned workspace, then (volume target, cell records)
    the int64 cell-gradient moments; refused if it does not fit."""
    from paper_2107_12672_b200 import _native as N
    vol, tf, prm = _descs(W=512, H=512)
    det = lambda v, m: lib.ddvr_deterministic_bytes(ctypes.byref(vol), v, ctypes.byref(prm),  # noqa
                                                    m)
    assert det(64, 1) == 32 * 32 * 64 * 24 and det(64, 2) == det(64, 3) == det(64, 1)
    assert det(64, 8) == 0 and det(64, 4) == 0             # no cell records: no int64 region
    prm.row0, prm.row1 = 100, 117                            # a 17-row band: 2 tile rows
    assert det(1, 1) == (32 * 2 * 24 + 255) // 256 * 256
    vol.cells = 32                                          # with cell records, the volume
    cells = (5 * 5 * 5 * 32 + 255) // 256 * 256             # target adds a 256-byte header +
    assert det(1, 8) == 256 + 2 * cells                     # the int64 moments (8 per record)
    assert det(1, 9) == det(1, 1) + det(1, 8)
    vol.cells = None
    vol, tf, prm = _descs()
    prm.flags = N.FLAG_DETERMINISTIC
    rc = lib.ddvr_adjoint(ctypes.byref(vol), ctypes.byref(tf), 16, 1, ctypes.byref(prm), 16,
                          None, 16, 1, None, None, 16, None, None, 0, None)
    assert rc == 2 and "deterministic" in lib.ddvr_last_error().decode()
    prm.flags = 1 << 20   # an unknown bit
    rc = lib.ddvr_adjoint(ctypes.byref(vol), ctypes.byref(tf), 16, 1, ctypes.byref(prm), 16,
                          None, 16, 1, None, None, 16, None, None, 0, None)
    assert rc == 1 and "flags" in lib.ddvr_last_error().decode()
    prm.flags = N.FLAG_RAY_SPLIT[2] | N.FLAG_RAY_SPLIT[8]   # two ray splits
    rc = lib.ddvr_adjoint(ctypes.byref(vol), ctypes.byref(tf), 16, 1, ctypes.byref(prm), 16,
                          None, 16, 1, None, None, 16, None, None, 0, None)
    assert rc == 1 and "RAY_SPLIT" in lib.ddvr_last_error().decode()


def test_band_tape_bytes_and_limits(lib):
    """ddvr_band_tape_bytes: 32-bit words per ray from the box diagonal / dt, for every
    pixel of every CTA, then the empty-brick map and the per-ray walk weights; a fused call whose tape would pass 2^32 words is refused
    before any CUDA work, and one without room for the tape asks for it."""
    import math
    from paper_2107_12672_b200 import _native as N
    vol, tf, prm = _descs(dt=0.01, W=512, H=512)
    words = math.ceil((math.floor(math.sqrt(3.0) / 0.01) + 3) / 32)
    assert lib.ddvr_band_tape_bytes(ctypes.byref(vol), 64, ctypes.byref(prm)) == \
        32 * 32 * 64 * 256 * words * 4 + 256 + 32 * 32 * 64 * 256 * 4
    # + the brick occupancy maps (1 brick, 256-aligned) + a float per ray (the walk weights
    # the march hands to the separate walk kernel)
    loss = ctypes.c_double(0)
    vol.cells = 32
    call = lambda v, p, nv, ws: lib.ddvr_forward_adjoint_l1(  # noqa: E731
        ctypes.byref(v), ctypes.byref(tf), 16, nv, ctypes.byref(p), 16, 8.0, 8, None, None,
        ctypes.addressof(loss), 16, None, None, None, 32, ws, None)
    prm.flags = N.FLAG_BAND_TAPE
    big_vol, _, big = _descs(dt=1e-3, W=4096, H=4096)
    big_vol.cells = 32
    big.flags = N.FLAG_BAND_TAPE
    assert call(big_vol, big, 64, 1 << 40) == 3 and "16 GiB" in lib.ddvr_last_error().decode()
    assert call(vol, prm, 1, 1 << 16) == 2 and "band tape" in lib.ddvr_last_error().decode()


def test_ray_split_choice(lib):
    """Segment-split rays (DDVR_FLAG_RAY_SPLIT_*): fused TF-target masks split by default
    only when the rays alone would not fill the GPU (C1's 16 K rays: 8 threads per ray;
    C2's 524 K: 1), camera / stepsize alone in two below four waves (C3), masks mixing
    them with TF or volume never; the flags force it."""
    from paper_2107_12672_b200 import _native as N
    TF, VOL, CAM = N.TARGET_BITS["tf"], N.TARGET_BITS["volume"], N.TARGET_BITS["camera"]
    split = lib.ddvr_ray_split
    assert split(TF | VOL, 128 * 128, 0) == 8          # C1
    assert split(TF, 8 * 256 * 256, 0) == 1            # C2
    assert split(TF, 40000, 0) == 4 and split(TF, 60000, 0) == 2
    for mask in (VOL, TF | CAM, VOL | CAM, TF | VOL | CAM):
        assert split(mask, 100, 0) == 1
        assert split(mask, 100, N.FLAG_RAY_SPLIT[4]) == 1
    for k, flag in N.FLAG_RAY_SPLIT.items():
        assert split(TF | VOL, 128 * 128, flag) == k
        assert split(TF, 10 ** 8, flag) == k
    # camera / stepsize alone: 2 lanes below 4 waves (forced: 2 or 4), never deterministic
    STEP = N.TARGET_BITS["stepsize"]
    for mask in (CAM, STEP, CAM | STEP):
        assert split(mask, 512 * 512, 0) == 2               # C3: 1.7 waves one thread per ray
        assert split(mask, 8 * 1024 * 1024, 0) == 1
        assert split(mask, 100, N.FLAG_RAY_SPLIT[1]) == 1
        assert split(mask, 100, N.FLAG_RAY_SPLIT[2]) == 2
        assert split(mask, 10 ** 6, N.FLAG_RAY_SPLIT[4]) == 4
        assert split(mask, 100, N.FLAG_RAY_SPLIT[8]) == 1
        assert split(mask, 100, N.FLAG_RAY_SPLIT[4] | N.FLAG_DETERMINISTIC) == 1
