"""Host-side API (no GPU): synthetic assets, build_crowd, camera / covariance / pose
records against the oracle, skinning KATs, memory model. Restates
/root/reference/proj/tests/test_avatar.cpp, test_crowd.cpp and acceptance.cpp criteria
that do not need the renderer."""
import math

import numpy as np
import pytest

import paper_2501_17792_b200 as P
from paper_2501_17792_b200.api import memory_report_cell
from oracle import orc


def make_scene(**kw):
    base = dict(template_count=1, level_counts=(60, 24, 8), motion_count=1, motion_frames=24, grid_rows=1,
                grid_cols=1, crowd_count=1, cam_pos=(0.0, 1.6, -3.0), cam_look=(0.0, 1.0, 5.0), width=160, height=90)
    base.update(kw)
    return P.Scene(P.SceneConfig(**base))


def test_template_level_counts_match_request():
    s = make_scene(template_seed_base=42, level_counts=P.api.LEVELS_PAPER)
    assert [s.level_view(0, l)["count"] for l in range(3)] == [202738, 12661, 3176]
    assert s.skeleton(0)["joint_count"] == 24


def test_template_deterministic_per_seed():
    a = make_scene(template_seed_base=7, level_counts=(400, 90), with_sh=True)
    b = make_scene(template_seed_base=7, level_counts=(400, 90), with_sh=True)
    c = make_scene(template_seed_base=8, level_counts=(400, 90))
    for l in range(2):
        va, vb = a.level_view(0, l), b.level_view(0, l)
        for k in ("means", "skin_weights", "colors", "sh", "cov6"):
            assert va[k].tobytes() == vb[k].tobytes()
    assert a.level_view(0, 0)["means"].tobytes() != c.level_view(0, 0)["means"].tobytes()


def test_template_invariants():
    s = make_scene(template_seed_base=3, level_counts=(100, 10), with_sh=True)
    v = s.level_view(0, 0)
    assert np.allclose(v["skin_weights"].sum(1), 1.0, atol=1e-5)
    assert (v["skin_indices"] < 24).all()
    assert np.allclose(np.linalg.norm(v["rotations"], axis=1), 1.0, atol=1e-6)
    assert (v["scales"] > 0).all() and ((v["opacities"] > 0) & (v["opacities"] <= 1)).all()
    assert v["sh"].shape == (100, 45) and np.abs(v["sh"]).max() <= 0.08


@pytest.mark.parametrize("counts", [(10, 20), (10, 10), (0,)])
def test_invalid_level_counts_rejected(counts):
    with pytest.raises(ValueError):
        make_scene(level_counts=counts)


def test_motion_loops_and_moves():
    s = make_scene(motion_frames=60)
    m = s.motion(0)
    assert m["frames"] == 60 and m["fps"] == 30.0
    q = m["data"][:, 4:].reshape(60, 24, 4)
    assert np.allclose(np.linalg.norm(q, axis=2), 1.0, atol=1e-5)
    assert (np.abs(q[10, :, 3] - 1.0) > 1e-4).any()


def test_build_crowd_benchmark_scale_population():
    s = P.Scene(P.SceneConfig(template_count=14, level_counts=(60, 24, 8), motion_count=15, motion_frames=24,
                              grid_rows=59, grid_cols=60, crowd_count=3500, crowd_seed=99))
    inst = s.instances
    assert len(inst) == 3500
    assert inst["x"].min() >= -0.26 and inst["x"].max() <= 59.26
    assert inst["z"].min() >= -0.26 and inst["z"].max() <= 58.26
    assert set(inst["template_id"].tolist()) == set(range(14))
    assert set(inst["motion_id"].tolist()) == set(range(15))
    assert (inst["phase_offset_s"] >= 0).all() and (inst["phase_offset_s"] < 24 / 30.0).all()


def test_build_crowd_single_cell_and_determinism():
    s = make_scene(crowd_seed=5)
    i = s.instances[0]
    assert abs(i["x"]) <= 0.25 and abs(i["z"]) <= 0.25
    a = make_scene(template_count=3, motion_count=2, grid_rows=8, grid_cols=8, crowd_count=64, crowd_seed=1234)
    b = make_scene(template_count=3, motion_count=2, grid_rows=8, grid_cols=8, crowd_count=64, crowd_seed=1234)
    c = make_scene(template_count=3, motion_count=2, grid_rows=8, grid_cols=8, crowd_count=64, crowd_seed=4321)
    assert a.instances.tobytes() == b.instances.tobytes()
    assert a.instances.tobytes() != c.instances.tobytes()


def test_build_crowd_capacity_error():
    with pytest.raises(ValueError):
        make_scene(grid_rows=3, grid_cols=3, crowd_count=10)


def test_host_camera_matches_oracle_bitwise():
    for pos, look, w, h in [((0.0, 1.6, -3.0), (0.0, 1.0, 5.0), 160, 90),
                            ((29.5, 1.6, -3.0), (29.5, 1.0, 5.0), 1920, 1080),
                            ((0.0, 0.95, -2.2), (0.0, 0.95, 0.0), 512, 512),
                            ((3.0, 10.0, 0.0), (3.0, -2.0, 0.01), 320, 240)]:
        s = make_scene(cam_pos=pos, cam_look=look, width=w, height=h)
        cam = s.camera_basis()
        w9 = np.zeros(9, np.float32)
        focal = orc.C.c_float()
        e, t = np.asarray(pos, np.float32), np.asarray(look, np.float32)
        orc.lib().orc_camera(e.ctypes.data, t.ctypes.data, 50.0, w, h, 0.1, w9.ctypes.data, orc.C.byref(focal), None)
        assert np.array(cam.world_to_view, np.float32).tobytes() == w9.tobytes()
        assert np.float32(cam.focal) == np.float32(focal.value)


def test_host_covariance_cache_matches_oracle_bitwise():
    s = make_scene(template_seed_base=9, level_counts=(2000, 300))
    o = orc.from_scene(s)
    for l in range(2):
        v = s.level_view(0, l)
        assert v["cov6"].tobytes() == o.level_cov(0, l, v["count"]).tobytes()


def test_host_pose_records_match_oracle_sample_pose():
    s = make_scene(template_count=2, motion_count=3, grid_rows=4, grid_cols=4, crowd_count=16, crowd_seed=77,
                   motion_frames=60)
    for t in (0.0, 0.37, 1.9, 12.345):
        tids, place, poses = s.sample_crowd(t)
        inst = s.instances
        for i in range(16):
            m = s.motion(int(inst["motion_id"][i]))
            ref = np.zeros(4 + 4 * 24, np.float32)
            orc.lib().orc_sample_pose(m["data"].ctypes.data, m["frames"], 24, m["fps"],
                                      np.float32(t) + inst["phase_offset_s"][i], 1, ref.ctypes.data)
            assert poses[i].tobytes() == ref.tobytes()
            assert place[i, 2] == np.float32(math.cos(np.float32(inst["yaw"][i]))) or \
                abs(place[i, 2] - math.cos(inst["yaw"][i])) < 1e-6


# ------------------------------------------------------- FK / LBS KATs (oracle, test_avatar.cpp)

def translation(t):
    m = np.eye(4, dtype=np.float32)
    m[:3, 3] = t
    return m.T.copy()  # column-major storage


def single_joint_scene(ibs, parents, means, idx, w):
    o = orc.OracleScene()
    o.add_template(np.asarray(parents, np.int16), np.asarray(ibs, np.float32).reshape(-1, 16))
    n = len(means)
    lv = {"count": n, "means": np.asarray(means, np.float32), "rotations": np.tile([0, 0, 0, 1], (n, 1)).astype(np.float32),
          "scales": np.full((n, 3), 0.1, np.float32), "opacities": np.ones(n, np.float32),
          "colors": np.ones((n, 3), np.float32), "skin_indices": np.asarray(idx, np.uint16),
          "skin_weights": np.asarray(w, np.float32), "sh": None}
    o.add_level(0, lv)
    return o


def fk(o, t, pose, root=None):
    J = (len(pose) - 4) // 4
    root = np.eye(4, dtype=np.float32) if root is None else root
    world = np.zeros((J, 16), np.float32)
    assert orc.lib().orc_forward_kinematics(o._h, t, np.ascontiguousarray(pose, np.float32).ctypes.data,
                                            np.ascontiguousarray(root, np.float32).ctypes.data, world.ctypes.data) == 0
    return world.reshape(J, 4, 4).transpose(0, 2, 1)  # -> row-major matrices


def skin(o, t, l, world_rm, n):
    world = np.ascontiguousarray(world_rm.transpose(0, 2, 1), np.float32)
    out = np.zeros((n, 3), np.float32)
    assert orc.lib().orc_skin_means(o._h, t, l, world.ctypes.data, out.ctypes.data) == 0
    return out


def test_fk_bind_pose_inverts_inverse_binds_and_lbs_identity():
    s = make_scene(template_seed_base=17, level_counts=(1200,))
    o = orc.from_scene(s)
    pose = np.zeros(4 + 96, np.float32)
    pose[7::4] = 1.0
    world = fk(o, 0, pose)
    ib = s.skeleton(0)["inverse_bind"].reshape(24, 4, 4).transpose(0, 2, 1)
    assert np.abs(world @ ib - np.eye(4)).max() < 1e-5
    v = s.level_view(0, 0)
    assert np.abs(skin(o, 0, 0, world, v["count"]) - v["means"]).max() < 1e-4


def test_fk_single_joint_z90_plus_translation():
    o = single_joint_scene([np.eye(4)], [-1], [[1, 0, 0]], [[0, 0, 0, 0]], [[1, 0, 0, 0]])
    pose = np.array([1, 0, 0, 0, *axis_angle_q(0.5 * 3.14159265, (0, 0, 1))], np.float32)
    world = fk(o, 0, pose)
    p = world[0] @ np.array([1, 0, 0, 1])
    assert np.allclose(p[:3], (1, 1, 0), atol=1e-5)
    posed = skin(o, 0, 0, world, 1)
    assert np.allclose(posed[0], (1, 1, 0), atol=1e-5)  # T(1,0,0) * Rz(90) * (1,0,0)


def axis_angle_q(angle, axis):
    axis = np.asarray(axis, np.float64) / np.linalg.norm(axis)
    return [*(math.sin(0.5 * angle) * axis), math.cos(0.5 * angle)]


def test_fk_two_joint_chain_composes():
    ibs = [np.eye(4, dtype=np.float32).T, translation((0, -1, 0))]
    o = single_joint_scene(ibs, [-1, 0], [[0, 0, 0]], [[0, 0, 0, 0]], [[1, 0, 0, 0]])
    q = axis_angle_q(0.25 * 3.14159265, (0, 0, 1))
    pose = np.array([0, 0, 0, 0, *q, *q], np.float32)
    world = fk(o, 0, pose)
    c, s = math.cos(math.pi / 4), math.sin(math.pi / 4)
    r45 = np.array([[c, -s, 0, 0], [s, c, 0, 0], [0, 0, 1, 0], [0, 0, 0, 1]])
    t1 = np.eye(4); t1[1, 3] = 1
    assert np.abs(world[1] - r45 @ t1 @ r45).max() < 1e-5
    assert np.abs(world[1][:3, :3] - (r45 @ r45)[:3, :3]).max() < 1e-5


def test_lbs_fifty_fifty_averages():
    ibs = [np.eye(4, dtype=np.float32), np.eye(4, dtype=np.float32)]
    o = single_joint_scene(ibs, [-1, 0], [[0, 0, 0]], [[0, 1, 0, 0]], [[0.5, 0.5, 0, 0]])
    world = np.stack([np.eye(4), np.eye(4)]).astype(np.float32)
    world[1, 2, 3] = 2.0
    posed = skin(o, 0, 0, world, 1)
    assert posed[0, 2] == pytest.approx(1.0, rel=1e-6) and posed[0, 0] == 0.0


def test_lbs_matches_double_precision_brute_force():
    rng = np.random.default_rng(31)
    for _ in range(8):
        J = 2 + int(rng.integers(23))
        n = 50 + int(rng.integers(951))
        parents = [-1] + [int(rng.integers(j)) for j in range(1, J)]
        ibs = [translation(-rng.uniform([-1, 0, -1], [1, 2, 1])) for _ in range(J)]
        means = rng.uniform([-1, 0, -1], [1, 2, 1], (n, 3))
        idx = rng.integers(0, J, (n, 4))
        w = rng.uniform(0, 1, (n, 4)).astype(np.float32)
        w /= w.sum(1, keepdims=True)
        o = single_joint_scene(ibs, parents, means, idx, w)
        q = rng.uniform(-1, 1, (J, 4))
        q /= np.linalg.norm(q, axis=1, keepdims=True)
        pose = np.concatenate([rng.uniform(-1, 1, 3), [0], q.ravel()]).astype(np.float32)
        world = fk(o, 0, pose)
        posed = skin(o, 0, 0, world, n)
        ibm = np.stack([np.asarray(m, np.float64).reshape(4, 4).T for m in ibs])
        Sm = world.astype(np.float64) @ ibm
        p4 = np.concatenate([means.astype(np.float32).astype(np.float64), np.ones((n, 1))], 1)
        ref = np.zeros((n, 3))
        for k in range(4):
            v = np.einsum("nij,nj->ni", Sm[idx[:, k]], p4)[:, :3]
            ref += w[:, k:k + 1].astype(np.float64) * v
        assert np.abs(posed - ref).max() < 1e-5


# ------------------------------------------------------------- memory model (test_crowd.cpp)

def test_memory_model_hand_arithmetic():
    r = memory_report_cell(100, 1000)
    assert r["resident_template_bytes"] == 80 * 1000
    assert r["naive_bytes"] == 80 * 1000 + 100 * 80 * 1000
    assert r["shared_bytes"] == 80 * 1000 + 100 * 12 * 1000
    assert r["savings_fraction"] == pytest.approx(1 - 1280 / 8080, rel=1e-12)
    one = memory_report_cell(1, 500)
    assert one["naive_bytes"] - one["shared_bytes"] == 68 * 500


def test_memory_model_marginal_slopes():
    for c in (1, 2, 100, 4999):
        lo, hi = memory_report_cell(c, 3176, 123456789), memory_report_cell(c + 1, 3176, 123456789)
        assert hi["naive_bytes"] - lo["naive_bytes"] == 80 * 3176
        assert hi["shared_bytes"] - lo["shared_bytes"] == 12 * 3176
    zero = memory_report_cell(0, 12661, 1 << 20)
    assert zero["shared_bytes"] == zero["naive_bytes"] == 1 << 20


def test_psnr_reference_definition():
    import paper_2501_17792_b200 as P

    rng = np.random.default_rng(3)
    a = rng.random((6, 7, 3), dtype=np.float32)
    assert P.psnr(a, a.copy()) == 99.0  # identical -> cap
    b = a.copy()
    b[2, 3, 1] += 0.25
    want = 10 * np.log10(1.0 / np.mean((a.astype(np.float64) - b.astype(np.float64)) ** 2))
    assert abs(P.psnr(a, b) - want) < 1e-4
    c = a.copy()
    c[0, 0, 0] += 1e-9  # below float resolution at that value? still capped only if identical
    assert P.psnr(a, c) <= 99.0
    with pytest.raises(ValueError):
        P.psnr(a, a[:, :-1])


def test_update_crowd_lod_matches_oracle():
    import paper_2501_17792_b200 as P
    from oracle import orc

    cfg, _ = P.baseline_config(2)
    cfg.lod_hysteresis = 0.5
    scene = P.Scene(cfg)
    o = orc.from_scene(scene)
    o.render(0.0, orc.settings(sh_colour=True), threads=4)
    scene.update_crowd()
    lods = scene.instances["active_lod"]
    assert np.array_equal(lods, o.lods(len(lods)))
    assert len(set(lods.tolist())) == 3  # all three levels present at config 2
    scene.update_crowd(forced_lod=7)  # clamped to the coarsest level
    assert np.all(scene.instances["active_lod"] == 2)
