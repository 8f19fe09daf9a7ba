"""CPU: the reference's file formats through libmdg's native readers/writers
(SURVEY §8f rank 4): raw volume + JSON sidecar (io_raw.cpp) and the MDT2
checkpoint (checkpoint.cpp).  The goldens under tests/golden/io/ were written
by the reference's own save_raw / save_checkpoint (oracle/gen_io_golden.sh);
re-writing what we load must reproduce them byte for byte."""
import os
import shutil

import numpy as np
import pytest

from paper_2403_16526_b200 import ops

GOLD = os.path.join(os.path.dirname(__file__), "golden", "io")


def g(name):
    return os.path.join(GOLD, name)


def same_bytes(a, b):
    return open(a, "rb").read() == open(b, "rb").read()


def test_raw_volume_roundtrip_is_byte_identical(tmp_path):
    v, sp = ops.load_raw_volume(g("vol.json"))
    assert v.shape == (3, 4, 5) and v.dtype == np.float32
    assert np.array_equal(v.ravel(), np.fromfile(g("vol.raw"), dtype="<f4"))
    assert sp == (1.0, float(np.float32(0.8)), 1.5)
    ops.save_raw_volume(tmp_path / "v", v, sp)
    assert same_bytes(tmp_path / "v.json", g("vol.json"))
    assert same_bytes(tmp_path / "v.raw", g("vol.raw"))


def test_raw_labels_roundtrip_is_byte_identical(tmp_path):
    lab, sp = ops.load_raw_labels(g("labels.json"))
    assert lab.dtype == np.int32 and lab.ravel()[3] == 65535
    assert np.array_equal(lab.ravel(), np.fromfile(g("labels.raw"), dtype="<u2").astype(np.int32))
    ops.save_raw_labels(tmp_path / "l", lab, sp)
    assert same_bytes(tmp_path / "l.json", g("labels.json"))
    assert same_bytes(tmp_path / "l.raw", g("labels.raw"))


def test_raw_field_roundtrip_is_byte_identical(tmp_path):
    f = ops.load_raw_field(g("field.json"))
    assert f.shape == (3, 3, 4, 5)
    ops.save_raw_field(tmp_path / "f", f)
    assert same_bytes(tmp_path / "f.json", g("field.json"))
    assert same_bytes(tmp_path / "f.raw", g("field.raw"))


@pytest.mark.parametrize("name", ["ckpt_a.mdt", "ckpt_b.mdt"])
def test_checkpoint_roundtrip_is_byte_identical(tmp_path, name):
    cfg, arrs, names = ops.load_checkpoint(g(name))
    assert len(arrs) == 75 and names[0] == "enc.l1.conv1.w" and names[-1] == "lvl4.reghead.b"
    ops.save_checkpoint(tmp_path / name, arrs, cfg)
    assert same_bytes(tmp_path / name, g(name))


def test_checkpoint_config_fields():
    cfg, _, _ = ops.load_checkpoint(g("ckpt_b.mdt"))
    assert cfg.base_channels == 1 and cfg.diffeomorphic == 1 and cfg.ss_steps == 5
    assert list(cfg.heads_per_level) == [3, 2, 2, 1, 1] and cfg.head_dim == 1
    assert cfg.leaky_slope == np.float32(0.1)


def test_small_preset_checkpoint_roundtrip(tmp_path):
    """init_model(small_preset, 42) -> save -> load is bitwise identical
    (io.hpp:40-41) and carries the reference's tensor names."""
    params = [t.numpy() for t in ops.init_model_native(42)]
    ops.save_checkpoint(tmp_path / "m.mdt", params)
    cfg, arrs, names = ops.load_checkpoint(tmp_path / "m.mdt")
    assert cfg.base_channels == 8 and list(cfg.heads_per_level) == [8, 4, 2, 1, 1]
    assert all(np.array_equal(a, p.ravel()) for a, p in zip(arrs, params))
    assert names[40:47] == ["lvl0.proj.w", "lvl0.proj.b", "lvl0.proj.ln_g", "lvl0.proj.ln_b",
                            "lvl0.bias_b", "lvl0.reghead.w", "lvl0.reghead.b"]


def test_sidecar_number_formatting(tmp_path):
    """The reference serializer's number layout (checked against nlohmann's
    own output for these values): shortest round-trip digits, integral values
    get '.0', exponent form once the decimal point is 5+ places in."""
    v = np.zeros((2, 2, 4), np.float32)
    ops.save_raw_volume(tmp_path / "x", v, (np.float32(1e-4), np.float32(1e-5), 123456.5))
    txt = open(tmp_path / "x.json").read()
    assert '"dims": [4,2,2]' in txt
    assert "    9.999999747378752e-05,\n" in txt
    assert "    9.999999747378752e-06,\n" in txt
    assert "    123456.5\n" in txt
    v2, sp = ops.load_raw_volume(tmp_path / "x.json")
    assert sp == (float(np.float32(1e-4)), float(np.float32(1e-5)), 123456.5)


def _copy(tmp_path, stem):
    for ext in (".json", ".raw"):
        shutil.copy(g(stem + ext), tmp_path / (stem + ext))
    return tmp_path / (stem + ".json")


def test_raw_errors(tmp_path):
    with pytest.raises(ops.ParseError, match="single-channel f32"):
        ops.load_raw_volume(g("labels.json"))
    with pytest.raises(ops.ParseError, match="3-channel f32"):
        ops.load_raw_field(g("vol.json"))
    with pytest.raises(ops.ParseError, match="u16"):
        ops.load_raw_labels(g("vol.json"))
    shutil.copy(g("vol.json"), tmp_path / "vol.txt")  # valid sidecar, wrong suffix
    with pytest.raises(ops.InvalidInput, match=".json sidecar"):
        ops.load_raw_volume(tmp_path / "vol.txt")
    with pytest.raises(ops.ParseError, match="cannot open"):
        ops.load_raw_volume(tmp_path / "missing.json")
    # payload length mismatch
    j = _copy(tmp_path, "vol")
    raw = open(tmp_path / "vol.raw", "rb").read()
    open(tmp_path / "vol.raw", "wb").write(raw[:-4])
    with pytest.raises(ops.ParseError, match="length mismatch"):
        ops.load_raw_volume(j)
    # non-finite voxel
    a = np.frombuffer(raw, dtype="<f4").copy()
    a[7] = np.nan
    a.tofile(tmp_path / "vol.raw")
    with pytest.raises(ops.ParseError, match="non-finite voxel"):
        ops.load_raw_volume(j)
    # sidecar problems
    open(j, "w").write('{"dims": [5,4,3], "dtype": "f32", "order": "zyx", "spacing": [1,1,1]}')
    with pytest.raises(ops.ParseError, match="xyz-row-major"):
        ops.load_raw_volume(j)
    open(j, "w").write('{"dims": [5,4], "dtype": "f32", "order": "xyz-row-major", "spacing": [1,1,1]}')
    with pytest.raises(ops.ParseError, match="3 entries"):
        ops.load_raw_volume(j)
    open(j, "w").write('{"dims": [5,4,3], "order": "xyz-row-major", "spacing": [1,1,1]}')
    with pytest.raises(ops.ParseError, match="missing field"):
        ops.load_raw_volume(j)
    open(j, "w").write('{"dims": [5,4,3], "dtype": "f32", ')
    with pytest.raises(ops.ParseError, match="invalid JSON"):
        ops.load_raw_volume(j)
    with pytest.raises(ops.InvalidInput, match="u16 range"):
        ops.save_raw_labels(tmp_path / "bad", np.full((2, 2, 2), 70000), (1, 1, 1))


def test_checkpoint_errors(tmp_path):
    blob = open(g("ckpt_a.mdt"), "rb").read()
    p = tmp_path / "c.mdt"
    open(p, "wb").write(b"MDT1" + blob[4:])
    with pytest.raises(ops.ParseError, match="magic"):
        ops.load_checkpoint(p)
    open(p, "wb").write(blob[:4] + (2).to_bytes(4, "little") + blob[8:])
    with pytest.raises(ops.ParseError, match="version"):
        ops.load_checkpoint(p)
    open(p, "wb").write(blob[: len(blob) - 100])
    with pytest.raises(ops.ParseError, match="truncated"):
        ops.load_checkpoint(p)
    # a tensor name that does not match the layout
    i = blob.index(b"enc.l1.conv1.b")
    open(p, "wb").write(blob[:i] + b"enc.l1.conv1.x" + blob[i + 14:])
    with pytest.raises(ops.ParseError, match="does not match expected"):
        ops.load_checkpoint(p)
    # config that fails ModelConfig::validate
    i = blob.index(b'"head_dim":2')
    open(p, "wb").write(blob[:i] + b'"head_dim":0' + blob[i + 12:])
    with pytest.raises(ops.InvalidInput, match="head_dim"):
        ops.load_checkpoint(p)
    with pytest.raises(ops.InvalidInput):
        ops.save_checkpoint(tmp_path / "x.mdt", [np.zeros(3)])


@pytest.mark.parametrize("name", ["img_u8", "img_i16", "img_f32"])
def test_nifti_matches_reference_loader(name):
    """load_nifti: voxels and spacing equal what the reference's loader returned
    for the same file (stored with save_raw by the golden generator)."""
    v, sp = ops.load_nifti(g(name + ".nii"))
    ve, spe = ops.load_raw_volume(g(name + "_expected.json"))
    assert v.shape == ve.shape and np.array_equal(v, ve) and sp == spe


def test_nifti_errors(tmp_path):
    blob = bytearray(open(g("img_i16.nii"), "rb").read())
    p = tmp_path / "x.nii"

    def expect(mut, match):
        b = bytearray(blob)
        mut(b)
        open(p, "wb").write(bytes(b))
        with pytest.raises(ops.ParseError, match=match):
            ops.load_nifti(p)

    expect(lambda b: b.__setitem__(slice(344, 348), b"ni1\0"), "magic")
    expect(lambda b: b.__setitem__(slice(0, 4), (349).to_bytes(4, "little")), "sizeof_hdr")
    expect(lambda b: b.__setitem__(slice(40, 42), (4).to_bytes(2, "little")), "dim\\[0\\] = 4")
    expect(lambda b: b.__setitem__(slice(70, 72), (8).to_bytes(2, "little")), "datatype 8")
    expect(lambda b: b.__setitem__(slice(72, 74), (8).to_bytes(2, "little")), "bitpix")
    expect(lambda b: b.__delitem__(slice(len(b) - 10, len(b))), "truncated NIfTI voxel")
    open(p, "wb").write(bytes(blob[:200]))
    with pytest.raises(ops.ParseError, match="truncated NIfTI header"):
        ops.load_nifti(p)
