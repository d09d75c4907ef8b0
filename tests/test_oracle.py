"""Pins the CPU oracle (oracle/orc.cpp) to the reference's own known-answer and property
tests. The reference ships no golden vectors and cannot be built here (Eigen 3.4 absent),
so these restatements of /root/reference/proj/tests/*.cpp are what make the oracle
trustworthy; tests/golden/ freezes a few of its frames as regression fixtures."""
import math

import numpy as np
import pytest

from oracle import orc
from oracle.orc import SPLAT_DTYPE

f32 = np.float32


def canonical(width=640, height=360, fov=50.0):
    return dict(eye=(0.0, 0.0, 0.0), target=(0.0, 0.0, 1.0), fov=fov, w=width, h=height, near=0.1)


def cov_of(q_xyzw, scale):
    out = np.zeros(9, dtype=np.float32)
    orc.lib().orc_build_covariance(np.asarray(q_xyzw, np.float32).ctypes.data,
                                   np.asarray(scale, np.float32).ctypes.data, out.ctypes.data)
    return out.reshape(3, 3)


def project(mean, cov, cam, color=(1, 1, 1), opacity=1.0):
    sp = orc.OrcSplat()
    m = np.asarray(mean, np.float32)
    c = np.ascontiguousarray(cov, np.float32)
    col = np.asarray(color, np.float32)
    e = np.asarray(cam["eye"], np.float32)
    t = np.asarray(cam["target"], np.float32)
    ok = orc.lib().orc_project(m.ctypes.data, c.ctypes.data, col.ctypes.data, opacity, e.ctypes.data, t.ctypes.data,
                               cam["fov"], cam["w"], cam["h"], cam["near"], orc.C.addressof(sp))
    return sp if ok else None


def camera(cam):
    w9 = np.zeros(9, np.float32)
    focal = orc.C.c_float()
    q = np.zeros(4, np.float32)
    e = np.asarray(cam["eye"], np.float32)
    t = np.asarray(cam["target"], np.float32)
    orc.lib().orc_camera(e.ctypes.data, t.ctypes.data, cam["fov"], cam["w"], cam["h"], cam["near"], w9.ctypes.data,
                         orc.C.byref(focal), q.ctypes.data)
    return w9.reshape(3, 3), focal.value, q


def axis_angle(angle, axis):
    axis = np.asarray(axis, np.float64)
    axis = axis / np.linalg.norm(axis)
    h = 0.5 * angle
    return np.array([*(math.sin(h) * axis), math.cos(h)], np.float32)


def quat_matrix(q):
    x, y, z, w = [float(v) for v in q]
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
                     [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
                     [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)]])


def unit_quats(rng, n):
    q = rng.uniform(-1, 1, size=(n, 4))
    return (q / np.linalg.norm(q, axis=1, keepdims=True)).astype(np.float32)


# ------------------------------------------------------------------ math (test_math.cpp)

def test_covariance_identity_exact():
    assert np.array_equal(cov_of((0, 0, 0, 1), (1, 1, 1)), np.eye(3, dtype=np.float32))


def test_covariance_axis_aligned():
    c = cov_of((0, 0, 0, 1), (2, 1, 1))
    assert np.allclose(np.diag(c), [4, 1, 1])
    assert abs(c[0, 1]) < 1e-7


def test_covariance_z90_permutes_axes():
    q = axis_angle(0.5 * 3.14159265, (0, 0, 1))
    c = cov_of(q, (2, 1, 1))
    r = quat_matrix(q)
    ref = r @ np.diag([4.0, 1.0, 1.0]) @ r.T
    assert np.abs(c - ref).max() < 1e-5
    assert np.allclose(np.diag(c), [1, 4, 1], rtol=1e-5)


def test_covariance_spectrum_rotation_invariant():
    rng = np.random.default_rng(11)
    for q in unit_quats(rng, 200):
        s = rng.uniform(0.1, 2.0, 3).astype(np.float32)
        c = cov_of(q, s)
        assert np.abs(c - c.T).max() < 1e-6
        ev = np.sort(np.linalg.eigvalsh(c.astype(np.float64)))
        assert np.allclose(ev, np.sort(s.astype(np.float64) ** 2), rtol=1e-4, atol=1e-4)
        r = quat_matrix(q)
        assert np.abs(c - r @ np.diag(s.astype(np.float64) ** 2) @ r.T).max() < 1e-5


def test_project_on_axis_lands_at_center():
    cam = canonical()
    _, f, _ = camera(cam)
    d, s = 4.0, 0.05
    sp = project((0, 0, d), np.eye(3) * s * s, cam)
    assert sp is not None
    assert sp.mean_px[0] == pytest.approx(320.0, rel=1e-4)
    assert sp.mean_px[1] == pytest.approx(180.0, rel=1e-4)
    expected = (f * s / d) ** 2 + 0.3
    assert sp.cov_xx == pytest.approx(expected, rel=1e-3)
    assert sp.cov_yy == pytest.approx(expected, rel=1e-3)
    assert sp.depth == pytest.approx(d, rel=1e-5)


def test_project_culls_behind_near_nan_and_offscreen():
    cam = canonical()
    cov = np.eye(3) * 0.01
    assert project((0, 0, -2.0), cov, cam) is None
    assert project((0, 0, 0.05), cov, cam) is None
    assert project((float("nan"), 0, 3.0), cov, cam) is None
    assert project((50.0, 0, 2.0), np.eye(3) * 1e-4, cam) is None


def test_project_mirror_symmetry():
    cam = canonical()
    _, _, qc = camera(cam)
    rwc = quat_matrix(qc)
    q = axis_angle(0.7, (1, 2, 0.5))
    s = (0.08, 0.03, 0.05)
    cs = np.array([0.8, 0.4, 5.0])
    a = project(rwc @ cs, cov_of(q, s), cam)
    qm = np.array([-q[0], q[1], -q[2], q[3]], np.float32)  # reflect rotation about x: (w, x, -y, -z)
    qm = np.array([q[0], -q[1], -q[2], q[3]], np.float32)
    b = project(rwc @ np.array([-cs[0], cs[1], cs[2]]), cov_of(qm, s), cam)
    assert a is not None and b is not None
    assert b.mean_px[0] == pytest.approx(cam["w"] - a.mean_px[0], rel=1e-4)
    assert b.mean_px[1] == pytest.approx(a.mean_px[1], rel=1e-4)
    assert b.cov_xx == pytest.approx(a.cov_xx, rel=1e-4)
    assert b.cov_yy == pytest.approx(a.cov_yy, rel=1e-4)
    assert b.cov_xy == pytest.approx(-a.cov_xy, rel=1e-4, abs=1e-6)


def test_project_matches_finite_differences():
    cam = canonical(1280, 720)
    W, f, _ = camera(cam)
    W = W.astype(np.float64)
    rng = np.random.default_rng(23)
    tested = 0
    while tested < 100:
        d = rng.uniform(2, 20)
        mean = np.array([rng.uniform(-0.4, 0.4) * d, rng.uniform(-0.2, 0.2) * d, d], np.float32)
        smax = 0.045 * d
        s = (rng.uniform(0.2, 1.0, 3) * smax).astype(np.float32)
        cov = cov_of(unit_quats(rng, 1)[0], s)
        sp = project(mean, cov, cam)
        if sp is None:
            continue
        tested += 1
        h = 1e-5 * (float(np.linalg.norm(mean)) + 1.0)

        def pix(p):
            t = W @ (p - np.zeros(3))
            return np.array([f * t[0] / t[2] + 0.5 * cam["w"], f * t[1] / t[2] + 0.5 * cam["h"]])

        J = np.zeros((2, 3))
        for ax in range(3):
            hi = mean.astype(np.float64).copy(); lo = hi.copy()
            hi[ax] += h; lo[ax] -= h
            J[:, ax] = (pix(hi) - pix(lo)) / (2 * h)
        fd = J @ cov.astype(np.float64) @ J.T + np.eye(2) * 0.3
        scale = max(abs(fd[0, 0]), abs(fd[1, 1]), 1.0)
        assert abs(sp.cov_xx - fd[0, 0]) / scale < 1e-3
        assert abs(sp.cov_yy - fd[1, 1]) / scale < 1e-3
        assert abs(sp.cov_xy - fd[0, 1]) / scale < 1e-3


def test_pixel_radius_scales_inverse_distance():
    cam = canonical(1280, 720)
    s = 0.03
    prev = None
    for d in (1.0, 2.0, 4.0, 8.0):
        sp = project((0, 0, d), np.eye(3) * s * s, cam)
        r = math.sqrt(sp.cov_xx - 0.3)
        if prev:
            assert abs(r - prev[0] * prev[1] / d) / (prev[0] * prev[1] / d) < 0.05
        prev = (r, d)


def test_projection_is_pure():
    cam = canonical()
    q = axis_angle(0.4, (0.2, 1, 0))
    cov = cov_of(q, (0.2, 0.1, 0.05))
    a = project((0.3, -0.2, 5.0), cov, cam)
    b = project((0.3, -0.2, 5.0), cov, cam)
    assert bytes(a) == bytes(b)


# ------------------------------------------------------------------- LoD (test_lod.cpp)

def lod(th, d, prev=None, band=0.0):
    t = np.asarray(th, np.float32)
    return orc.lib().orc_select_lod(t.ctypes.data, len(t), band, d, -1 if prev is None else prev)


def test_lod_canonical_distances_and_boundaries():
    th = (5.0, 10.0)
    assert [lod(th, d) for d in (4.9, 7.0, 12.0, 0.0, 10.0, 5.0)] == [0, 1, 2, 0, 2, 1]


def test_lod_hysteresis_shifts_boundary():
    th = (5.0, 10.0)
    assert lod(th, 5.3, 0, 1.0) == 0
    assert lod(th, 5.6, 0, 1.0) == 1
    assert lod(th, 4.7, 1, 1.0) == 1
    assert lod(th, 4.4, 1, 1.0) == 0


def test_lod_matches_interval_scan():
    th = (2.0, 5.0, 10.0, 30.0)
    rng = np.random.default_rng(3)
    ds = np.concatenate([rng.uniform(0, 40, 10000).astype(np.float32), np.asarray(th, np.float32)])
    for d in ds:
        assert lod(th, float(d)) == sum(1 for t in th if d >= np.float32(t))


def test_lod_monotone_and_no_oscillation():
    th = (5.0, 10.0)
    for prev in (None, 0, 1, 2):
        band = 1.0 if prev is not None else 0.0
        last = 0
        for d in np.arange(0, 20, 0.01, dtype=np.float32):
            lv = lod(th, float(d), prev, band)
            assert lv >= last
            last = lv
    for b in th:
        lo, hi = b - 0.25, b + 0.25
        level = lod(th, hi, None, 1.0)
        first = level
        for i in range(100):
            level = lod(th, lo if i % 2 else hi, level, 1.0)
            assert level == first


# ----------------------------------------------------------- raster (test_renderer.cpp)

def splat(mean, cov_d, depth, color, opacity, inst, gauss, w, h):
    s = np.zeros(1, SPLAT_DTYPE)[0]
    s["mean_px"] = mean
    s["cov_xx"] = s["cov_yy"] = cov_d
    s["depth"] = depth
    s["color"] = color
    s["opacity"] = opacity
    s["instance_id"], s["gaussian_index"] = inst, gauss
    rx = f32(3) * np.sqrt(f32(cov_d))
    s["rect"] = [max(0, int(math.floor(f32(mean[0]) - rx))), max(0, int(math.floor(f32(mean[1]) - rx))),
                 min(w, int(math.floor(f32(mean[0]) + rx)) + 1), min(h, int(math.floor(f32(mean[1]) + rx)) + 1)]
    return s


def raster(sp, w, h, st, threads=0, naive=False):
    sp = np.ascontiguousarray(sp, SPLAT_DTYPE)
    rgb = np.zeros((h, w, 3), np.float32)
    T = np.zeros((h, w), np.float32)
    p = sp.ctypes.data if len(sp) else None
    if naive:
        orc.lib().orc_naive_rasterize(p, len(sp), w, h, orc.C.byref(st), rgb.ctypes.data, T.ctypes.data)
    else:
        assert orc.lib().orc_rasterize(p, len(sp), w, h, orc.C.byref(st), threads, rgb.ctypes.data, T.ctypes.data) == 0
    return rgb, T


def sort_splats(sp):
    sp = np.ascontiguousarray(sp, SPLAT_DTYPE).copy()
    if len(sp):
        orc.lib().orc_sort_splats(sp.ctypes.data, len(sp))
    return sp


def random_frame(rng, w, h, count):
    """oracles.hpp:227-255 random splat frame."""
    out = []
    for i in range(count):
        mx, my = rng.uniform(-8, w + 8), rng.uniform(-8, h + 8)
        th = rng.uniform(0, 6.2831853)
        l0, l1 = rng.uniform(0.5, 60), rng.uniform(0.5, 60)
        c, s_ = math.cos(th), math.sin(th)
        sp = np.zeros(1, SPLAT_DTYPE)[0]
        sp["mean_px"] = (mx, my)
        sp["cov_xx"] = f32(c * c * l0 + s_ * s_ * l1 + 0.3)
        sp["cov_yy"] = f32(s_ * s_ * l0 + c * c * l1 + 0.3)
        sp["cov_xy"] = f32(c * s_ * (l0 - l1))
        sp["depth"] = rng.uniform(0.2, 50)
        sp["color"] = rng.uniform(0, 1, 3)
        sp["opacity"] = rng.uniform(0.05, 1.0)
        sp["instance_id"] = rng.integers(0, 8)
        sp["gaussian_index"] = i
        mxf, myf = f32(sp["mean_px"][0]), f32(sp["mean_px"][1])
        rx, ry = f32(3) * np.sqrt(sp["cov_xx"]), f32(3) * np.sqrt(sp["cov_yy"])
        r = [max(0, int(math.floor(mxf - rx))), max(0, int(math.floor(myf - ry))),
             min(w, int(math.floor(mxf + rx)) + 1), min(h, int(math.floor(myf + ry)) + 1)]
        if r[0] >= r[2] or r[1] >= r[3]:
            continue
        sp["rect"] = r
        out.append(sp)
    return np.array(out, SPLAT_DTYPE)


def test_raster_background_only():
    st = orc.settings(background=(0.2, 0.4, 0.6))
    rgb, T = raster(np.zeros(0, SPLAT_DTYPE), 33, 17, st)
    assert np.all(rgb[..., 0] == f32(0.2)) and np.all(rgb[..., 1] == f32(0.4)) and np.all(rgb[..., 2] == f32(0.6))
    assert np.all(T == 1.0)


def test_raster_clamped_opaque_white():
    sp = np.array([splat((16.5, 16.5), 9.0, 1.0, (1, 1, 1), 1.0, 0, 0, 32, 32)])
    rgb, _ = raster(sp, 32, 32, orc.settings())
    assert np.allclose(rgb[16, 16], 0.99, rtol=1e-6)


def test_raster_red_over_blue():
    sp = np.array([splat((8.5, 8.5), 16.0, 1.0, (1, 0, 0), 0.5, 0, 0, 16, 16),
                   splat((8.5, 8.5), 16.0, 2.0, (0, 0, 1), 0.5, 0, 1, 16, 16)])
    rgb, _ = raster(sort_splats(sp), 16, 16, orc.settings(background=(1, 1, 1)))
    assert np.allclose(rgb[8, 8], (0.75, 0.25, 0.5), rtol=1e-6)


def test_sort_matches_stable_comparison_sort_with_ties():
    rng = np.random.default_rng(19)
    fr = random_frame(rng, 128, 128, 300)
    fr["depth"][1::8] = fr["depth"][0::8][: len(fr["depth"][1::8])]
    ref = sorted(range(len(fr)), key=lambda i: (fr["depth"][i], fr["instance_id"][i], fr["gaussian_index"][i]))
    got = sort_splats(fr)
    assert np.array_equal(got["instance_id"], fr["instance_id"][ref])
    assert np.array_equal(got["gaussian_index"], fr["gaussian_index"][ref])


def test_tiled_raster_bit_identical_to_naive():
    rng = np.random.default_rng(101)
    for _ in range(8):
        w, h = 96 + int(rng.integers(64)), 64 + int(rng.integers(48))
        fr = sort_splats(random_frame(rng, w, h, 80 + int(rng.integers(421))))
        st = orc.settings(background=tuple(rng.uniform(0, 1, 3)), tile_size=1 + int(rng.integers(40)))
        a, at = raster(fr, w, h, st)
        b, bt = raster(fr, w, h, st, naive=True)
        assert a.tobytes() == b.tobytes() and at.tobytes() == bt.tobytes()


def test_raster_weights_plus_transmittance_is_one():
    rng = np.random.default_rng(7)
    fr = sort_splats(random_frame(rng, 80, 60, 250))
    st = orc.settings()
    _, T = raster(fr, 80, 60, st)
    cut = f32(1) / f32(255)
    for py in range(0, 60, 3):
        for px in range(0, 80, 3):
            t, wsum = 1.0, 0.0
            for s in fr:
                x0, y0, x1, y1 = s["rect"]
                if not (x0 <= px < x1 and y0 <= py < y1):
                    continue
                det = s["cov_xx"] * s["cov_yy"] - s["cov_xy"] * s["cov_xy"]
                inv = f32(1) / det
                a, b, c = s["cov_yy"] * inv, -s["cov_xy"] * inv, s["cov_xx"] * inv
                dx, dy = f32(px) + f32(0.5) - s["mean_px"][0], f32(py) + f32(0.5) - s["mean_px"][1]
                power = f32(-0.5) * (a * dx * dx + c * dy * dy) - b * dx * dy
                if power < np.log(cut / s["opacity"]):
                    continue
                alpha = min(float(s["opacity"]) * math.exp(float(power)), 0.99)
                wsum += t * alpha
                t *= 1 - alpha
                if t < 1e-4:
                    break
            assert wsum + t == pytest.approx(1.0, rel=1e-5)
            assert T[py, px] == pytest.approx(t, rel=1e-4, abs=1e-6)


def test_raster_convex_hull():
    rng = np.random.default_rng(57)
    fr = sort_splats(random_frame(rng, 64, 48, 200))
    rgb, _ = raster(fr, 64, 48, orc.settings(background=(0.3, 0.3, 0.3)))
    assert rgb.min() >= 0.0 and rgb.max() <= 1.0 + 1e-5


def test_raster_thread_count_invariant():
    rng = np.random.default_rng(5)
    fr = sort_splats(random_frame(rng, 120, 90, 400))
    outs = [raster(fr, 120, 90, orc.settings(), threads=t)[0].tobytes() for t in (1, 4, 8)]
    assert outs[0] == outs[1] == outs[2]


# --------------------------------------------------------- poses (test_avatar.cpp)

def sample_pose(clip, frames, joints, fps, t, wrap=True):
    out = np.zeros(4 + 4 * joints, np.float32)
    assert orc.lib().orc_sample_pose(clip.ctypes.data, frames, joints, fps, t, int(wrap), out.ctypes.data) == 0
    return out


def quat_angle(a, b):
    """Eigen angularDistance: 2 atan2(|vec(a^-1 b)|, |w(a^-1 b)|)."""
    ax, ay, az, aw = (float(v) for v in a)
    bx, by, bz, bw = (float(v) for v in b)
    ax, ay, az = -ax, -ay, -az  # conjugate
    w = aw * bw - ax * bx - ay * by - az * bz
    x = aw * bx + ax * bw + ay * bz - az * by
    y = aw * by - ax * bz + ay * bw + az * bx
    z = aw * bz + ax * by - ay * bx + az * bw
    return 2 * math.atan2(math.sqrt(x * x + y * y + z * z), abs(w))


def test_sample_pose_halfway_slerp_is_45_degrees():
    clip = np.zeros((2, 8), np.float32)
    clip[0, 4:8] = (0, 0, 0, 1)
    clip[1, 4:8] = axis_angle(0.5 * 3.14159265, (0, 0, 1))
    mid = sample_pose(clip, 2, 1, 1.0, 0.5, wrap=False)
    assert quat_angle(mid[4:8], axis_angle(0.25 * 3.14159265, (0, 0, 1))) < 1e-5


def test_sample_pose_clamp_holds_last_frame():
    rng = np.random.default_rng(8)
    clip = np.zeros((20, 8), np.float32)
    clip[:, :3] = rng.uniform(-1, 1, (20, 3))
    clip[:, 4:8] = unit_quats(rng, 20)
    a = sample_pose(clip, 20, 1, 10.0, 100.0, wrap=False)
    assert np.array_equal(a[:3], clip[-1, :3])


def test_sample_pose_time_zero_is_frame_zero():
    rng = np.random.default_rng(3)
    clip = np.zeros((16, 8), np.float32)
    clip[:, :3] = rng.uniform(-1, 1, (16, 3))
    clip[:, 4:8] = unit_quats(rng, 16)
    p = sample_pose(clip, 16, 1, 30.0, 0.0)
    assert np.array_equal(p[:3], clip[0, :3])
    assert quat_angle(p[4:8], clip[0, 4:8]) < 1e-6


def test_sample_pose_empty_clip_rejected():
    out = np.zeros(8, np.float32)
    assert orc.lib().orc_sample_pose(out.ctypes.data, 0, 1, 30.0, 0.0, 1, out.ctypes.data) != 0
