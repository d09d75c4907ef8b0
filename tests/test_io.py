"""GSAT / GSMO asset files (§8f row 2), mirroring the reference's io tests
(test_io.cpp:36-199): byte-identical round trips, bit-exact floats, typed failures,
truncation naming its section at the reference's byte offsets, and the v2 SH extension.
CPU only (host library)."""
from __future__ import annotations

import numpy as np
import pytest

import paper_2501_17792_b200 as P
from paper_2501_17792_b200 import FormatError


def scene(levels=(40, 10), sh=False, templates=1, motions=1, frames=6):
    cfg = P.SceneConfig(template_count=templates, template_seed_base=6, level_counts=levels, with_sh=sh,
                        motion_count=motions, motion_frames=frames, grid_rows=2, grid_cols=2, crowd_count=4)
    return P.Scene(cfg)


def level_arrays(s, t):
    out = []
    for l in range(s.level_count(t)):
        v = s.level_view(t, l)
        out.append({k: np.array(v[k]) for k in ("means", "rotations", "scales", "opacities", "colors",
                                                  "skin_indices", "skin_weights", "cov6", "sh")})
    return out


def test_gsat_roundtrip_resave_is_byte_identical(tmp_path):
    s = scene(levels=(40, 10, 3))
    p1, p2 = tmp_path / "a.gsat", tmp_path / "b.gsat"
    s.save_template(0, p1)
    t = s.load_template(p1)
    assert t == 1
    s.save_template(1, p2)
    assert p1.read_bytes() == p2.read_bytes()
    a, b = level_arrays(s, 0), level_arrays(s, 1)
    assert len(a) == len(b) == 3
    for la, lb in zip(a, b):
        for k in la:
            assert la[k].tobytes() == lb[k].tobytes(), k  # bit-exact, incl. the derived covariance
    sk0, sk1 = s.skeleton(0), s.skeleton(1)
    assert np.array_equal(sk0["parents"], sk1["parents"])
    assert sk0["inverse_bind"].tobytes() == sk1["inverse_bind"].tobytes()


def test_gsat_v1_layout_offsets(tmp_path):
    s = scene(levels=(10,))
    p = tmp_path / "t.gsat"
    s.save_template(0, p)
    b = p.read_bytes()
    J, n = 24, 10
    assert b[:4] == b"GSAT" and int.from_bytes(b[4:8], "little") == 1
    assert int.from_bytes(b[8:10], "little") == J and b[10] == 1
    count_off = 11 + 2 * J + 64 * J
    assert int.from_bytes(b[count_off:count_off + 4], "little") == n
    lv = s.level_view(0, 0)
    means = np.frombuffer(b[count_off + 4:count_off + 4 + 12 * n], dtype="<f4").reshape(n, 3)
    assert means.tobytes() == np.array(lv["means"], dtype=np.float32).tobytes()
    rot = np.frombuffer(b[count_off + 4 + 12 * n:count_off + 4 + 28 * n], dtype="<f4").reshape(n, 4)
    q = np.array(lv["rotations"], dtype=np.float32)  # x, y, z, w in memory; w, x, y, z on disk
    assert rot.tobytes() == q[:, [3, 0, 1, 2]].tobytes()
    per = 12 + 16 + 12 + 4 + 12 + 8 + 16
    assert len(b) == count_off + 4 + per * n


def test_gsat_v2_carries_sh(tmp_path):
    s = scene(levels=(30, 8), sh=True)
    p = tmp_path / "sh.gsat"
    s.save_template(0, p)
    assert int.from_bytes(p.read_bytes()[4:8], "little") == 2
    s.load_template(p)
    a, b = level_arrays(s, 0), level_arrays(s, 1)
    for la, lb in zip(a, b):
        assert la["sh"].size == lb["sh"].size > 0
        assert la["sh"].tobytes() == lb["sh"].tobytes()


def test_gsmo_roundtrip_bit_exact(tmp_path):
    s = scene(frames=7)
    p1, p2 = tmp_path / "m.gsmo", tmp_path / "m2.gsmo"
    s.save_motion(0, p1)
    m = s.load_motion(p1)
    s.save_motion(m, p2)
    assert p1.read_bytes() == p2.read_bytes()
    a, b = s.motion(0), s.motion(m)
    assert a["fps"] == b["fps"] and a["frames"] == b["frames"] == 7
    assert a["data"].tobytes() == b["data"].tobytes()


def test_gsmo_one_frame_identity_clip(tmp_path):
    s = scene()
    data = np.zeros((1, 4 + 4 * 4), dtype=np.float32)
    data[0, 4 + 3::4] = 1.0  # w = 1
    s.set_motion(1, 30.0, data, 4)
    p = tmp_path / "id.gsmo"
    s.save_motion(1, p)
    m = s.load_motion(p)
    mo = s.motion(m)
    assert mo["frames"] == 1 and mo["joints"] == 4


def test_bad_magic_and_version(tmp_path):
    s = scene()
    p = tmp_path / "x.gsat"
    s.save_template(0, p)
    b = bytearray(p.read_bytes())
    bad = tmp_path / "bad.gsat"
    bad.write_bytes(b"XXXX" + bytes(b[4:]))
    with pytest.raises(FormatError) as e:
        s.load_template(bad)
    assert e.value.kind == "BadMagic"
    b[4:8] = (7).to_bytes(4, "little")
    bad.write_bytes(bytes(b))
    with pytest.raises(FormatError) as e:
        s.load_template(bad)
    assert e.value.kind == "VersionMismatch"
    mp = tmp_path / "x.gsmo"
    s.save_motion(0, mp)
    with pytest.raises(FormatError) as e:
        s.load_motion(p)  # a template is not a motion
    assert e.value.kind == "BadMagic"


@pytest.mark.parametrize("keep,section", [
    (2, "magic"), (11 - 1, "header"), (11 + 2 * 24 - 3, "parents"),
    (11 + 2 * 24 + 64 * 24 - 10, "inverse_bind"), (11 + 2 * 24 + 64 * 24 + 4 + 11, "level 0 means")])
def test_truncation_names_the_section(tmp_path, keep, section):
    s = scene(levels=(40, 10))
    p = tmp_path / "trunc.gsat"
    s.save_template(0, p)
    p.write_bytes(p.read_bytes()[:keep])
    with pytest.raises(FormatError) as e:
        s.load_template(p)
    assert e.value.kind == "Truncated" and section in str(e.value)


def test_invariant_violations_are_typed(tmp_path):
    s = scene()
    mp = tmp_path / "badfps.gsmo"
    s.save_motion(0, mp)
    b = bytearray(mp.read_bytes())
    b[8:12] = bytes(4)  # fps = 0
    mp.write_bytes(bytes(b))
    with pytest.raises(FormatError) as e:
        s.load_motion(mp)
    assert e.value.kind == "InvariantViolation"
    tp = tmp_path / "badquat.gsat"
    s2 = scene(levels=(10,))
    s2.save_template(0, tp)
    tb = bytearray(tp.read_bytes())
    rot = 11 + 2 * 24 + 64 * 24 + 4 + 12 * 10
    tb[rot:rot + 16] = bytes(16)  # zero quaternion
    tp.write_bytes(bytes(tb))
    with pytest.raises(FormatError) as e:
        s2.load_template(tp)
    assert e.value.kind == "InvariantViolation"
    tb2 = bytearray(tp.read_bytes())
    tp.write_bytes(bytes(tb2) + b"\x00")
    with pytest.raises(FormatError):
        s2.load_template(tp)


def test_missing_file_is_io_error(tmp_path):
    s = scene()
    with pytest.raises(FormatError) as e:
        s.load_template(tmp_path / "missing.gsat")
    assert e.value.kind == "IoError"
    with pytest.raises(FormatError) as e:
        s.save_motion(0, tmp_path / "no" / "such" / "dir.gsmo")
    assert e.value.kind == "IoError"


def test_load_replaces_slot_and_crowd_still_samples(tmp_path):
    s = scene(templates=2, levels=(20, 5))
    p = tmp_path / "t1.gsat"
    s.save_template(1, p)
    assert s.load_template(p, 0) == 0  # slot 0 now holds template 1's data
    a, b = level_arrays(s, 0), level_arrays(s, 1)
    assert a[0]["means"].tobytes() == b[0]["means"].tobytes()
    tids, place, poses = s.sample_crowd(0.25)
    assert len(tids) == 4 and np.isfinite(poses).all()
