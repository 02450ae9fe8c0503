"""Pins for the CPU oracle: checks against what the paper and mathematics fix, never
against the oracle itself (closed forms, the paper's worked example, library
routines for special cases, brute force, finite differences).  CPU only."""
import json
import math
import os

import numpy as np
import pytest
from scipy.spatial.transform import Rotation

import oracle
from synth import scenes as S

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _one_gaussian(mean, quat, scale, opac, color, viewmat=None, K=None, W=64, H=64):
    return dict(means=np.array([mean], np.float32), quats=np.array([quat], np.float32),
                scales=np.array([scale], np.float32), opacities=np.array([opac], np.float32),
                colors=np.array([color], np.float32), sh_degree=-1,
                viewmats=(np.eye(4, dtype=np.float32) if viewmat is None else np.asarray(viewmat, np.float32))[None],
                Ks=np.array([K if K is not None else [[64, 0, 32], [0, 64, 32], [0, 0, 1]]], np.float32),
                width=W, height=H)


def _splat2d(means2d, conics, opac, rgb, depths, radii, C=1):
    """A hand-built projected set for camera 0 (bypasses projection)."""
    n = len(means2d)
    return dict(radii=np.array(radii, np.int32).reshape(C, n, 2),
                mean2d_f=np.array(means2d, np.float32).reshape(C, n, 2),
                depth_f=np.array(depths, np.float32).reshape(C, n),
                dec=np.concatenate([np.array(conics, np.float32).reshape(C, n, 3),
                                    np.array(opac, np.float32).reshape(C, n, 1)], axis=-1),
                mean2d=np.array(means2d, np.float64).reshape(C, n, 2),
                conic=np.array(conics, np.float64).reshape(C, n, 3),
                opac_eff=np.array(opac, np.float64).reshape(C, n),
                rgb=np.array(rgb, np.float64).reshape(C, n, 3))


# --------------------------------------------------------------------------- F1
class TestQuaternion:
    """P:778-782 (Hamilton, (w,x,y,z)); S:38-40 examples."""

    def test_identity_and_pi_about_z(self, oracle_lib):
        assert np.allclose(oracle.quat_to_rotmat([1, 0, 0, 0]), np.eye(3), atol=0)
        assert np.allclose(oracle.quat_to_rotmat([0, 0, 0, 1]), np.diag([-1.0, -1.0, 1.0]), atol=1e-15)
        assert np.allclose(oracle.quat_to_rotmat([2, 0, 0, 0]), np.eye(3), atol=0)

    def test_matches_scipy_hamilton(self, oracle_lib):
        rng = np.random.default_rng(1)
        for _ in range(200):
            q = rng.normal(size=4)
            R = oracle.quat_to_rotmat(q)
            Rs = Rotation.from_quat([q[1], q[2], q[3], q[0]]).as_matrix()   # scipy is scalar-last
            assert np.allclose(R, Rs, atol=1e-12)
            assert np.allclose(R.T @ R, np.eye(3), atol=1e-12)
            assert abs(np.linalg.det(R) - 1) < 1e-12
            assert np.allclose(oracle.quat_to_rotmat(3.7 * q), R, atol=1e-12)


# --------------------------------------------------------------------------- F1-F10
def _cov3d_ref(q, s):
    R = Rotation.from_quat([q[1], q[2], q[3], q[0]]).as_matrix()
    return R @ np.diag(np.asarray(s, np.float64) ** 2) @ R.T


def _pinhole(t, fx, fy, cx, cy):
    return np.array([fx * t[0] / t[2] + cx, fy * t[1] / t[2] + cy])


def _fd_jacobian(t, fx, fy, cx, cy, h=1e-6):
    J = np.zeros((2, 3))
    for k in range(3):
        e = np.zeros(3); e[k] = h * max(1.0, abs(t[k]))
        J[:, k] = (_pinhole(t + e, fx, fy, cx, cy) - _pinhole(t - e, fx, fy, cx, cy)) / (2 * e[k])
    return J


class TestProjection:
    def test_fig1_golden(self, oracle_lib):
        g = json.load(open(os.path.join(GOLD, "fig1.json")))
        sc = S.fig1_scene(scale=g["inputs"]["scale"])
        o = oracle.Options(sh_degree=-1)
        p = oracle.project(sc, o)
        ex = g["expected"]
        assert p["mean2d_f"][0, 0].tolist() == ex["mean2d"]
        assert p["depth_f"][0, 0] == np.float32(ex["depth"])
        assert p["radii"][0, 0].tolist() == [ex["radius"], ex["radius"]]
        cov = np.linalg.inv(np.array([[p["conic"][0, 0, 0], p["conic"][0, 0, 1]],
                                      [p["conic"][0, 0, 1], p["conic"][0, 0, 2]]]))
        assert np.allclose(np.diag(cov), ex["cov2d_blurred_diag"], rtol=1e-7)  # z = f32(0.01)
        keys, ids, offs = oracle.isect(p, 1, 1, 240, 240, o)
        assert len(keys) == ex["n_intersections"]

    def test_pixel_mapping_examples(self, oracle_lib):
        """on-axis -> (cx, cy); t=(2,0,2), fx=100, cx=50 -> mu'_x = 150."""
        o = oracle.Options(sh_degree=-1, fov_clamp=0)
        sc = _one_gaussian([2, 0, 2], [1, 0, 0, 0], [0.01] * 3, 0.5, [1, 1, 1],
                           K=[[100, 0, 50], [0, 100, 50], [0, 0, 1]], W=400, H=100)
        p = oracle.project(sc, o)
        assert p["mean2d"][0, 0, 0] == 150.0 and p["mean2d_f"][0, 0, 0] == 150.0
        sc = _one_gaussian([0, 0, 3.3], [1, 0, 0, 0], [0.01] * 3, 0.5, [1, 1, 1])
        p = oracle.project(sc, o)
        assert np.allclose(p["mean2d"][0, 0], [32, 32], atol=0)

    @pytest.mark.parametrize("seed", range(8))
    def test_cov2d_equals_fd_jacobian_sandwich(self, oracle_lib, seed):
        """Sigma' = J W Sigma W^T J^T (Fig. P:423) with J the FD Jacobian of the
        pinhole map and Sigma = R S S^T R^T from scipy."""
        rng = np.random.default_rng(seed)
        q = rng.normal(size=4); s = np.exp(rng.uniform(-3, -1, 3))
        Rc = Rotation.random(random_state=seed).as_matrix()
        mu = rng.uniform(-0.3, 0.3, 3)
        Vm = np.eye(4); Vm[:3, :3] = Rc
        t_want = np.array([rng.uniform(-0.4, 0.4), rng.uniform(-0.4, 0.4), rng.uniform(2, 4)])
        Vm[:3, 3] = t_want - Rc @ mu
        K = [[80.0, 0, 40.0], [0, 90.0, 30.0], [0, 0, 1]]
        sc = _one_gaussian(mu, q, s, 0.5, [1, 1, 1], viewmat=Vm, K=K, W=80, H=60)
        o = oracle.Options(sh_degree=-1, fov_clamp=0)
        p = oracle.project(sc, o)
        # reference in f64 from the f32 inputs the oracle saw
        mu32 = sc["means"][0].astype(np.float64); Vm32 = sc["viewmats"][0].astype(np.float64)
        t = Vm32[:3, :3] @ mu32 + Vm32[:3, 3]
        J = _fd_jacobian(t, 80.0, 90.0, 40.0, 30.0)
        Sig = _cov3d_ref(sc["quats"][0].astype(np.float64), sc["scales"][0].astype(np.float64))
        Sp = J @ Vm32[:3, :3] @ Sig @ Vm32[:3, :3].T @ J.T + 0.3 * np.eye(2)
        cov = np.linalg.inv(np.array([[p["conic"][0, 0, 0], p["conic"][0, 0, 1]],
                                      [p["conic"][0, 0, 1], p["conic"][0, 0, 2]]]))
        assert np.allclose(cov, Sp, rtol=1e-6, atol=1e-9)
        assert np.allclose(p["mean2d"][0, 0], _pinhole(t, 80.0, 90.0, 40.0, 30.0), rtol=1e-12)
        assert p["depth"][0, 0] == pytest.approx(t[2], rel=1e-12)

    def test_cov2d_on_axis_diag(self, oracle_lib):
        """Sigma_c = diag(a,b,c) on axis -> Sigma' = diag(a f^2/z^2, b f^2/z^2) (+0.3)."""
        o = oracle.Options(sh_degree=-1, fov_clamp=0)
        z, f = 2.0, 100.0
        s = [0.02, 0.05, 0.3]
        sc = _one_gaussian([0, 0, z], [1, 0, 0, 0], s, 0.5, [1, 1, 1],
                           K=[[f, 0, 32], [0, f, 32], [0, 0, 1]])
        p = oracle.project(sc, o)
        s32 = np.float32(s).astype(np.float64)
        want = np.diag([s32[0] ** 2 * f * f / (z * z) + 0.3, s32[1] ** 2 * f * f / (z * z) + 0.3])
        cov = np.linalg.inv(np.array([[p["conic"][0, 0, 0], p["conic"][0, 0, 1]],
                                      [p["conic"][0, 0, 1], p["conic"][0, 0, 2]]]))
        assert np.allclose(cov, want, rtol=1e-12, atol=1e-12)
        # isotropic radii: r = ceil(3 sigma)
        assert p["radii"][0, 0].tolist() == [math.ceil(3 * math.sqrt(want[0, 0])), math.ceil(3 * math.sqrt(want[1, 1]))]

    def test_antialias_compensation(self, oracle_lib):
        """A.4: Sigma' = I, s = 0.3 -> comp = sqrt(1/1.69) = 1/1.3; in (0,1];
        non-increasing in s; classic mode -> 1."""
        # f/z = 1 and sigma = 1 gives Sigma' = I exactly
        sc = _one_gaussian([0, 0, 1.0], [1, 0, 0, 0], [1.0, 1.0, 1.0], 0.8, [1, 1, 1],
                           K=[[1, 0, 32], [0, 1, 32], [0, 0, 1]])
        p = oracle.project(sc, oracle.Options(sh_degree=-1, antialiased=1, fov_clamp=0))
        assert p["comp"][0, 0] == pytest.approx(1 / 1.3, abs=1e-12)
        assert p["opac_eff"][0, 0] == pytest.approx(float(np.float32(0.8)) / 1.3, abs=1e-12)
        p = oracle.project(sc, oracle.Options(sh_degree=-1, antialiased=0, fov_clamp=0))
        assert p["comp"][0, 0] == 1.0
        prev = 1.0
        for eps in [0.0, 0.1, 0.3, 1.0, 3.0]:
            c = oracle.project(sc, oracle.Options(sh_degree=-1, antialiased=1, fov_clamp=0, eps2d=eps))["comp"][0, 0]
            assert 0 < c <= 1 and c <= prev + 1e-15
            prev = c

    def test_near_plane_and_culls(self, oracle_lib):
        """Q18 (depth == near renders; Fig. 1), S:158-160 culls."""
        o = oracle.Options(sh_degree=-1)
        sc = _one_gaussian([0, 0, -1], [1, 0, 0, 0], [0.1] * 3, 0.5, [1, 1, 1])
        assert oracle.project(sc, o)["radii"][0, 0].tolist() == [0, 0]
        sc = _one_gaussian([0, 0, 0.0099], [1, 0, 0, 0], [0.001] * 3, 0.5, [1, 1, 1])
        assert oracle.project(sc, o)["radii"][0, 0].tolist() == [0, 0]
        # far off screen: mu' = (-100,-100) on a 32x32 image, tiny radius
        sc = _one_gaussian([-1.32, -1.32, 1.0], [1, 0, 0, 0], [0.001] * 3, 0.5, [1, 1, 1],
                           K=[[100, 0, 32], [0, 100, 32], [0, 0, 1]], W=32, H=32)
        assert oracle.project(sc, o)["radii"][0, 0].tolist() == [0, 0]
        # zero quaternion -> culled, not an error (Q31)
        sc = _one_gaussian([0, 0, 2], [0, 0, 0, 0], [0.1] * 3, 0.5, [1, 1, 1])
        assert oracle.project(sc, o)["radii"][0, 0].tolist() == [0, 0]

    def test_fov_clamp_only_affects_J(self, oracle_lib):
        """Q27: the clamp changes Sigma' of an off-frustum splat but never mu'."""
        sc = _one_gaussian([2.5, 0.3, 1.0], [1, 0, 0, 0], [0.5, 0.2, 0.3], 0.5, [1, 1, 1],
                           K=[[20, 0, 32], [0, 20, 32], [0, 0, 1]], W=64, H=64)
        a = oracle.project(sc, oracle.Options(sh_degree=-1, fov_clamp=0))
        b = oracle.project(sc, oracle.Options(sh_degree=-1, fov_clamp=1))
        assert np.array_equal(a["mean2d"], b["mean2d"])
        assert a["radii"][0, 0, 0] > 0 and b["radii"][0, 0, 0] > 0
        assert not np.allclose(a["conic"], b["conic"])


    def test_fov_clamp_sigma_equals_fd_jacobian_at_clamped_point(self, oracle_lib):
        """Q27: for a splat deep inside the clamp, Sigma' is the sandwich
        with the pinhole Jacobian evaluated at the CLAMPED camera point
        t_c = (t_z u_c, t_z v_c, t_z), u_c = the widened-frustum limit; FD Jacobian of the
        pinhole map there, 3D covariance from scipy's rotation."""
        rng = np.random.default_rng(3)
        f, W, H = 40.0, 64, 48
        cx, cy = 30.0, 26.0
        lim_xp = (W - cx) / f + 0.3 * (W / 2) / f
        lim_xn = cx / f + 0.3 * (W / 2) / f
        lim_yp = (H - cy) / f + 0.3 * (H / 2) / f
        lim_yn = cy / f + 0.3 * (H / 2) / f
        n_checked = 0
        for k in range(12):
            z = rng.uniform(1.0, 3.0)
            u = rng.choice([-1, 1]) * rng.uniform(1.1, 1.6)          # far outside [-0.99, 1.2]
            v = rng.uniform(-0.3, 0.3) if k % 2 else rng.choice([-1, 1]) * rng.uniform(1.1, 1.5)
            q = rng.normal(size=4)
            s = rng.uniform(0.4, 1.2, 3)
            sc = _one_gaussian([u * z, v * z, z], q, s, 0.5, [1, 1, 1],
                               K=[[f, 0, cx], [0, f, cy], [0, 0, 1]], W=W, H=H)
            p = oracle.project(sc, oracle.Options(sh_degree=-1, fov_clamp=1))
            if p["radii"][0, 0, 0] == 0:
                continue
            m32 = sc["means"][0].astype(np.float64)
            uc = min(lim_xp, max(-lim_xn, m32[0] / m32[2]))
            vc = min(lim_yp, max(-lim_yn, m32[1] / m32[2]))
            assert uc != m32[0] / m32[2]                        # the clamp is active
            tc = np.array([m32[2] * uc, m32[2] * vc, m32[2]])
            J = _fd_jacobian(tc, f, f, cx, cy)
            Sig = _cov3d_ref(sc["quats"][0].astype(np.float64), sc["scales"][0].astype(np.float64))
            want = J @ Sig @ J.T + 0.3 * np.eye(2)
            Y = p["conic"][0, 0]
            got = np.linalg.inv(np.array([[Y[0], Y[1]], [Y[1], Y[2]]]))
            assert np.allclose(got, want, rtol=1e-6, atol=1e-6), (got, want)
            # mu' is never clamped (Q27)
            assert np.allclose(p["mean2d"][0, 0], _pinhole(m32, f, f, cx, cy), rtol=1e-12)
            n_checked += 1
        assert n_checked >= 6

    def test_bbox_mode1_square_lambda_max(self, oracle_lib):
        """Q12 option bbox_mode 1: r_x = r_y = ceil(3 sqrt(lambda_max)) of
        Sigma'+sI.  Closed form on a rotated anisotropic splat on the optical axis: Sigma' =
        (f/z)^2 R2 diag(sx^2, sy^2) R2^T, so lambda_max = (f/z)^2 max(sx, sy)^2 + 0.3 for every
        rotation angle about the view axis, while the per-axis box (mode 0) changes with it."""
        f, z = 100.0, 4.0
        sx, sy, sz = 0.3, 0.1, 0.05
        seen0 = set()
        for th in [0.0, 0.35, 0.6, 1.1, 2.0]:
            q = [math.cos(th / 2), 0, 0, math.sin(th / 2)]
            sc = _one_gaussian([0, 0, z], q, [sx, sy, sz], 0.5, [1, 1, 1],
                               K=[[f, 0, 50], [0, f, 50], [0, 0, 1]], W=100, H=100)
            p1 = oracle.project(sc, oracle.Options(sh_degree=-1, bbox_mode=1))
            s32 = float(np.float32(sx))
            lam = (f / z) ** 2 * s32 ** 2 + 0.3
            assert p1["radii"][0, 0].tolist() == [math.ceil(3 * math.sqrt(lam))] * 2 == [23, 23]
            p0 = oracle.project(sc, oracle.Options(sh_degree=-1, bbox_mode=0))
            c, s_ = math.cos(th), math.sin(th)
            sxx = (f / z) ** 2 * (c * c * s32 ** 2 + s_ * s_ * float(np.float32(sy)) ** 2) + 0.3
            syy = (f / z) ** 2 * (s_ * s_ * s32 ** 2 + c * c * float(np.float32(sy)) ** 2) + 0.3
            assert p0["radii"][0, 0].tolist() == [math.ceil(3 * math.sqrt(sxx)), math.ceil(3 * math.sqrt(syy))]
            seen0.add(tuple(p0["radii"][0, 0].tolist()))
        assert len(seen0) >= 3

    def test_bbox_mode1_equals_eigvalsh(self, oracle_lib):
        """bbox_mode 1 on random poses: r = ceil(3 sqrt(max eigenvalue)) of the fp64 Sigma'+sI
        (numpy eigvalsh), skipping the few whose 3 sqrt(lambda) lies within 1e-4 of an integer
        (the radii are an fp32 key-path decision, Q28)."""
        sc = S.tiny_scene(21, N=300, width=96, height=80, sh_degree=-1)
        p = oracle.project(sc, oracle.Options(sh_degree=-1, bbox_mode=1))
        vis = p["radii"][0, :, 0] > 0
        assert vis.sum() > 200
        checked = 0
        for n in np.nonzero(vis)[0]:
            Y = p["conic"][0, n]
            cov = np.linalg.inv(np.array([[Y[0], Y[1]], [Y[1], Y[2]]]))
            r = 3 * math.sqrt(np.linalg.eigvalsh(cov).max())
            if abs(r - round(r)) < 1e-4:
                continue
            assert p["radii"][0, n].tolist() == [math.ceil(r)] * 2
            checked += 1
        assert checked > 200


# --------------------------------------------------------------------------- SH
class TestSH:
    def test_orthonormal_quadrature(self, oracle_lib):
        """Real SH up to degree 3 are orthonormal on S^2 (Gauss-Legendre x uniform phi)."""
        nt, nphi = 24, 48
        x, w = np.polynomial.legendre.leggauss(nt)
        G = np.zeros((16, 16))
        for ct, wt in zip(x, w):
            st = math.sqrt(1 - ct * ct)
            for k in range(nphi):
                ph = 2 * math.pi * k / nphi
                d = (st * math.cos(ph), st * math.sin(ph), ct)
                Y = oracle.sh_basis(3, d)
                G += np.outer(Y, Y) * wt * (2 * math.pi / nphi)
        assert np.allclose(G, np.eye(16), atol=1e-12)

    def test_signs_real_sh_condon_shortley(self, oracle_lib):
        """Q22 pinned to a library routine: the 16 basis functions (signs included) are the
        real spherical harmonics built from scipy's complex Y_l^m (Condon-Shortley phase
        included) as sqrt(2) Im Y_l^|m| (m < 0), Y_l^0, sqrt(2) Re Y_l^m (m > 0), index
        l^2 + l + m -- the convention whose degree-1 terms are (-C1 y, C1 z, -C1 x)."""
        from scipy.special import sph_harm_y
        rng = np.random.default_rng(22)
        for _ in range(200):
            d = rng.normal(size=3)
            d /= np.linalg.norm(d)
            theta, phi = math.acos(d[2]), math.atan2(d[1], d[0])
            ref = np.zeros(16)
            for l in range(4):
                for m in range(-l, l + 1):
                    y = sph_harm_y(l, abs(m), theta, phi)
                    ref[l * l + l + m] = (math.sqrt(2) * y.imag if m < 0 else
                                          (y.real if m == 0 else math.sqrt(2) * y.real))
            assert np.allclose(oracle.sh_basis(3, d), ref, rtol=0, atol=1e-12)

    def test_degree0_colour(self, oracle_lib):
        """colour = 0.5 + 0.2820948 * dc."""
        sc = S.tiny_scene(3, N=10, sh_degree=0)
        p = oracle.project(sc, oracle.Options(sh_degree=0))
        vis = p["radii"][0, :, 0] > 0
        raw = 0.5 + 0.28209479177387814 * sc["colors"][:, 0, :].astype(np.float64)
        assert np.allclose(p["rgb"][0][vis], np.maximum(raw[vis], 0), atol=1e-15)

    def test_basis_gradient_fd(self, oracle_lib):
        rng = np.random.default_rng(5)
        for _ in range(20):
            d = rng.normal(size=3)
            g = oracle.sh_basis_grad(3, d)
            for k in range(3):
                e = np.zeros(3); e[k] = 1e-6
                fd = (oracle.sh_basis(3, d + e) - oracle.sh_basis(3, d - e)) / 2e-6
                assert np.allclose(g[:, k], fd, rtol=1e-7, atol=1e-8)


# --------------------------------------------------------------------------- I1-I4
class TestIsect:
    def test_one_tile_and_four_tiles(self, oracle_lib):
        """radius 3 inside a tile -> 1 tile; centred on a 4-tile corner -> 4."""
        o = oracle.Options()
        p = _splat2d([[8.0, 8.0]], [[1, 0, 1]], [0.5], [[1, 1, 1]], [1.0], [[3, 3]])
        k, i, off = oracle.isect(p, 1, 1, 64, 64, o)
        assert len(k) == 1 and np.diff(off)[0] == 1
        p = _splat2d([[16.0, 16.0]], [[1, 0, 1]], [0.5], [[1, 1, 1]], [1.0], [[3, 3]])
        k, i, off = oracle.isect(p, 1, 1, 64, 64, o)
        assert len(k) == 4 and sorted(np.nonzero(np.diff(off))[0].tolist()) == [0, 1, 4, 5]

    def test_random_scene_invariants(self, oracle_lib):
        """Sort order unique and non-decreasing, every (tile, id) inside the 3-sigma
        tile rectangle, ranges sum to M, each bin's ids sorted by depth."""
        sc = S.tiny_scene(11, N=300, width=100, height=70, sh_degree=0, views=2)
        o = oracle.Options(sh_degree=0)
        p = oracle.project(sc, o)
        C, N, W, H = 2, 300, 100, 70
        keys, ids, off = oracle.isect(p, C, N, W, H, o)
        TX, TY = 7, 5
        B = 6
        assert np.all(np.diff(keys.astype(np.float64)) >= 0)
        assert off[-1] == len(keys) and np.all(np.diff(off) >= 0)
        tot = 0
        for cam in range(C):
            for t in range(TX * TY):
                seg = slice(off[cam * TX * TY + t], off[cam * TX * TY + t + 1])
                gids = ids[seg]
                assert np.all(gids // N == cam)
                n = gids % N
                d = p["depth_f"][cam, n]
                assert np.all(np.diff(d) >= 0)
                assert np.all((keys[seg] >> np.uint64(32 + B)) == cam)
                assert np.all(((keys[seg] >> np.uint64(32)) & np.uint64((1 << B) - 1)) == t)
                tx, ty = t % TX, t // TX
                for g in n:
                    mx, my = p["mean2d_f"][cam, g]
                    rx, ry = p["radii"][cam, g]
                    # the tile's pixel square [16tx, 16tx+16) intersects [mx-rx, mx+rx] (closed)
                    assert mx - rx <= 16 * tx + 16 and mx + rx >= 16 * tx
                    assert my - ry <= 16 * ty + 16 and my + ry >= 16 * ty
                tot += len(n)
        assert tot == len(keys)
        # completeness: brute force over all tiles with the half-open rectangle definition
        cnt = 0
        for cam in range(C):
            for n in range(N):
                rx, ry = p["radii"][cam, n]
                if rx == 0:
                    continue
                mx, my = p["mean2d_f"][cam, n]
                for ty in range(TY):
                    for tx in range(TX):
                        x0 = min(max(math.floor(np.float32(mx - np.float32(rx)) / 16), 0), TX)
                        x1 = min(max(math.ceil(np.float32(mx + np.float32(rx)) / 16), 0), TX)
                        y0 = min(max(math.floor(np.float32(my - np.float32(ry)) / 16), 0), TY)
                        y1 = min(max(math.ceil(np.float32(my + np.float32(ry)) / 16), 0), TY)
                        cnt += int(x0 <= tx < x1 and y0 <= ty < y1)
        assert cnt == len(keys)


# --------------------------------------------------------------------------- R1-R3
class TestComposite:
    gold = json.load(open(os.path.join(GOLD, "composite_examples.json")))

    def _render(self, p, W=16, H=16, bg=None, **kw):
        o = oracle.Options(**kw)
        return oracle.render_fwd(p, 1, p["mean2d"].shape[1], W, H, o, backgrounds=bg)

    def test_two_splats(self, oracle_lib):
        g = self.gold["two_splats"]
        # alpha = o at the splat centre (Delta = 0): pixel (5,5) centre is (5.5, 5.5)
        p = _splat2d([[5.5, 5.5], [5.5, 5.5]], [[1, 0, 1], [1, 0, 1]], g["alphas"], g["colors"],
                     [1.0, 2.0], [[3, 3], [3, 3]])
        r = self._render(p)
        assert np.allclose(r["rgb"][0, 5, 5], g["expected_rgb"], atol=1e-15)
        assert r["alpha"][0, 5, 5] == pytest.approx(g["expected_alpha"], abs=1e-15)
        # order is by depth, not by index: swap depths -> green in front
        p2 = _splat2d([[5.5, 5.5], [5.5, 5.5]], [[1, 0, 1], [1, 0, 1]], g["alphas"], g["colors"],
                      [2.0, 1.0], [[3, 3], [3, 3]])
        assert np.allclose(self._render(p2)["rgb"][0, 5, 5], [0.25, 0.5, 0], atol=1e-15)

    def test_termination(self, oracle_lib):
        g = self.gold["termination"]
        n = len(g["alphas"])
        p = _splat2d([[5.5, 5.5]] * n, [[1, 0, 1]] * n, g["alphas"], [[1, 1, 1]] * n,
                     [1.0, 2.0, 3.0, 4.0], [[3, 3]] * n)
        r = self._render(p)
        assert r["T"][0, 5, 5] == pytest.approx(g["expected_T_final"], rel=1e-12)
        assert r["last_gid"][0, 5, 5] == g["expected_last_index"]
        assert r["ncontrib"][0, 5, 5] == 3

    def test_saturation_and_half_alpha(self, oracle_lib):
        g = self.gold["saturation"]
        p = _splat2d([[5.5, 5.5]], [[1, 0, 1]], [g["opacity"]], [[1, 1, 1]], [1.0], [[3, 3]])
        assert self._render(p)["alpha"][0, 5, 5] == pytest.approx(g["expected_alpha"], abs=1e-15)
        # |Delta| = sqrt(2 ln 2) along x with unit conic -> alpha = 0.5
        d = math.sqrt(2 * math.log(2))
        p = _splat2d([[5.5 + d, 5.5]], [[1, 0, 1]], [1.0], [[1, 1, 1]], [1.0], [[3, 3]])
        assert self._render(p)["alpha"][0, 5, 5] == pytest.approx(0.5, abs=1e-12)

    def test_isotropic_alpha_profile(self, oracle_lib):
        """alpha = o exp(-k^2 / (2 sigma^2)) along a row for isotropic Sigma' = sigma^2 I."""
        sig2 = 7.3
        p = _splat2d([[8.5, 8.5]], [[1 / sig2, 0, 1 / sig2]], [0.7], [[1, 1, 1]], [1.0], [[12, 12]])
        r = self._render(p, W=32, H=32)
        for k in range(0, 8):
            want = 0.7 * math.exp(-k * k / (2 * sig2))
            got = r["alpha"][0, 8, 8 + k]
            assert got == (pytest.approx(want, abs=1e-15) if want >= 1 / 255 else 0.0)

    def test_background_and_zero_opacity(self, oracle_lib):
        """Q25 and S:238: all opacities 0 -> background everywhere; alpha + T = 1."""
        sc = S.tiny_scene(2, N=50, sh_degree=0)
        sc["opacities"][:] = 0
        o = oracle.Options(sh_degree=0)
        p = oracle.project(sc, o)
        bg = np.array([[0.1, 0.2, 0.3]])
        r = oracle.render_fwd(p, 1, 50, 64, 64, o, backgrounds=bg)
        assert np.allclose(r["rgb"], bg[0], atol=0)
        sc = S.tiny_scene(2, N=50, sh_degree=0)
        p = oracle.project(sc, o)
        r = oracle.render_fwd(p, 1, 50, 64, 64, o, backgrounds=bg)
        assert np.allclose(r["alpha"] + r["T"], 1.0, atol=1e-15)
        assert np.all((r["T"] > 0) & (r["T"] <= 1))

    def test_permutation_invariance(self, oracle_lib):
        """permuting Gaussians at distinct depths does not change the image."""
        sc = S.tiny_scene(4, N=80, sh_degree=0)
        o = oracle.Options(sh_degree=0)
        r1 = oracle.render_fwd(oracle.project(sc, o), 1, 80, 64, 64, o)
        perm = np.random.default_rng(0).permutation(80)
        sc2 = dict(sc)
        for k in ["means", "quats", "scales", "opacities", "colors"]:
            sc2[k] = sc[k][perm]
        r2 = oracle.render_fwd(oracle.project(sc2, o), 1, 80, 64, 64, o)
        assert np.array_equal(r1["rgb"], r2["rgb"])

    def test_tiled_equals_global_walk(self, oracle_lib):
        """Brute force with tiles: per-tile lists from the sorted intersections,
        composited in numpy per tile, equal the oracle's global-sort walk."""
        sc = S.tiny_scene(6, N=120, width=72, height=40, sh_degree=0, views=2)
        o = oracle.Options(sh_degree=0)
        C, N, W, H = 2, 120, 72, 40
        p = oracle.project(sc, o)
        keys, ids, off = oracle.isect(p, C, N, W, H, o)
        r = oracle.render_fwd(p, C, N, W, H, o)
        TX, TY = 5, 3
        img = np.zeros((C, H, W, 3)); Tf = np.ones((C, H, W))
        for cam in range(C):
            for t in range(TX * TY):
                tx, ty = t % TX, t // TX
                ys, xs = np.mgrid[ty * 16:min(ty * 16 + 16, H), tx * 16:min(tx * 16 + 16, W)]
                px, py = xs + 0.5, ys + 0.5
                T = np.ones(px.shape); col = np.zeros(px.shape + (3,)); done = np.zeros(px.shape, bool)
                for g in ids[off[cam * TX * TY + t]:off[cam * TX * TY + t + 1]]:
                    cam_, n = divmod(int(g), N)
                    dx = p["mean2d"][cam_, n, 0] - px; dy = p["mean2d"][cam_, n, 1] - py
                    A, Bc, Cc = p["conic"][cam_, n]
                    sig = 0.5 * (A * dx * dx + Cc * dy * dy) + Bc * dx * dy
                    a = np.minimum(0.99, p["opac_eff"][cam_, n] * np.exp(-sig))
                    use = (~done) & (sig >= 0) & (a >= 1 / 255)
                    nT = T * (1 - a)
                    stop = use & (nT <= 1e-4)
                    done |= stop
                    use &= ~stop
                    col += np.where(use[..., None], p["rgb"][cam_, n] * (a * T)[..., None], 0)
                    T = np.where(use, nT, T)
                img[cam, ys, xs] = col; Tf[cam, ys, xs] = T
        assert np.allclose(r["rgb"], img, atol=1e-12)
        assert np.allclose(r["T"], Tf, atol=1e-12)


# --------------------------------------------------------------------------- B1-B6 and P1-P9
def _clean_scene(seed, N=24, W=32, H=32, sh_degree=1, views=1, antialiased=0, max_tries=400):
    """Rejection-sample a small scene with no pixel within 1e-3 (relative) of the alpha_min,
    alpha_max or T_min decisions (SURVEY 8c FD protocol)."""
    o = oracle.Options(sh_degree=sh_degree, antialiased=antialiased, amb_rel_floor=2e-3)
    for k in range(max_tries):
        sc = S.tiny_scene(seed * 1000 + k, N=N, width=W, height=H, sh_degree=sh_degree, views=views)
        sc["scales"] *= 1.5
        p = oracle.project(sc, o)
        r = oracle.render_fwd(p, views, N, W, H, o)
        if not r["ambig"].any() and (p["radii"][..., 0] > 0).sum() >= N // 2:
            return sc, o
    raise RuntimeError("no clean scene")


def _loss(sc, o, v_img, v_a, bg=None, v_d=None, v_e=None):
    C, N = sc["viewmats"].shape[0], sc["means"].shape[0]
    p = oracle.project(sc, o)
    r = oracle.render_fwd(p, C, N, sc["width"], sc["height"], o, backgrounds=bg)
    _, ids, offs = oracle.isect(p, C, N, sc["width"], sc["height"], o)
    l = float((r["rgb"] * v_img).sum() + (r["alpha"] * v_a).sum())
    if v_d is not None:
        l += float((r["depth"] * v_d).sum())
    if v_e is not None:
        l += float((r["depth_exp"] * v_e).sum())
    return l, (ids, offs)


class TestBackward:
    gold = json.load(open(os.path.join(GOLD, "composite_examples.json")))

    def test_single_and_two_splat_examples(self, oracle_lib):
        o = oracle.Options()
        p = _splat2d([[5.5, 5.5]], [[1, 0, 1]], [0.5], [[0.3, 0.4, 0.5]], [1.0], [[3, 3]])
        v = np.zeros((1, 16, 16, 3)); v[0, 5, 5] = 1.0
        b = oracle.render_bwd(p, 1, 1, 16, 16, o, v)
        assert np.allclose(b["v2d"][0, 0, 5:8], self.gold["backward_single"]["expected_v_rgb"], atol=1e-15)
        g = self.gold["two_splats"]
        p = _splat2d([[5.5, 5.5], [5.5, 5.5]], [[1, 0, 1], [1, 0, 1]], g["alphas"], g["colors"],
                     [1.0, 2.0], [[3, 3], [3, 3]])
        v = np.zeros((1, 16, 16, 3)); v[0, 5, 5, 1] = 1.0     # L = C_green
        b = oracle.render_bwd(p, 1, 2, 16, 16, o, v)
        # at Delta = 0, alpha = o_eff, so dL/do_eff = dC_g/dalpha_1
        assert b["v2d"][0, 0, 8] == pytest.approx(self.gold["backward_two"]["expected_dCg_dalpha1"], abs=1e-15)

    def test_clamped_alpha_has_no_opacity_gradient(self, oracle_lib):
        """Q24: o_eff e^-sigma > alpha_max -> d alpha / d o_eff = 0."""
        o = oracle.Options()
        p = _splat2d([[5.5, 5.5]], [[1, 0, 1]], [1.0], [[0.3, 0.4, 0.5]], [1.0], [[3, 3]])
        v = np.zeros((1, 16, 16, 3)); v[0, 5, 5] = 1.0
        b = oracle.render_bwd(p, 1, 1, 16, 16, o, v)
        assert b["v2d"][0, 0, 8] == 0.0 and b["v2d"][0, 0, 0] == 0.0

    @pytest.mark.parametrize("seed,bg", [(0, False), (1, True), (2, False)])
    def test_render_bwd_matches_fd(self, oracle_lib, seed, bg):
        """Every 2D gradient (mean2d, conic, rgb, opac_eff) = central FD of the f64 render
        of the loss <v_img, C> + <v_alpha, alpha> (Q25, Q26)."""
        sc, o = _clean_scene(seed, sh_degree=0)
        C, N, W, H = 1, sc["means"].shape[0], sc["width"], sc["height"]
        p = oracle.project(sc, o)
        rng = np.random.default_rng(seed)
        v_img = rng.normal(size=(C, H, W, 3)); v_a = rng.normal(size=(C, H, W))
        bgs = np.array([[0.2, 0.5, 0.9]]) if bg else None
        b = oracle.render_bwd(p, C, N, W, H, o, v_img, v_a, backgrounds=bgs)
        assert b["T_replay_err"] < 1e-12
        def L(pp):
            r = oracle.render_fwd(pp, C, N, W, H, o, backgrounds=bgs)
            return (r["rgb"] * v_img).sum() + (r["alpha"] * v_a).sum()
        fields = [("mean2d", 0, 2), ("conic", 2, 3), ("rgb", 5, 3), ("opac_eff", 8, 1)]
        vis = np.nonzero(p["radii"][0, :, 0] > 0)[0]
        checked = 0
        for n in vis:
            for name, off, k in fields:
                for j in range(k):
                    h = 1e-6
                    pp = {kk: vv.copy() for kk, vv in p.items()}
                    arr = pp[name].reshape(C, N, -1)
                    arr[0, n, j] += h; lp = L(pp)
                    arr[0, n, j] -= 2 * h; lm = L(pp)
                    fd = (lp - lm) / (2 * h)
                    an = b["v2d"][0, n, off + j]
                    assert abs(an - fd) <= 1e-5 * abs(fd) + 1e-7 * (1 + b["a2d"][0, n, off + j]), (name, n, j, an, fd)
                    checked += 1
        assert checked > 50

    @pytest.mark.parametrize("seed,sh,aa", [(0, 0, 0), (1, 1, 0), (2, 3, 0), (3, 1, 1), (4, 3, 1)])
    def test_full_chain_matches_fd(self, oracle_lib, seed, sh, aa):
        """End-to-end: d loss / d(means, quats, scales, opacities, colours) from
        project_bwd(render_bwd(...)) equals central FD over the f32 inputs (exact steps)."""
        sc, o = _clean_scene(seed + 10, sh_degree=sh, antialiased=aa, views=2)
        C, N, W, H = 2, sc["means"].shape[0], sc["width"], sc["height"]
        rng = np.random.default_rng(seed)
        v_img = rng.normal(size=(C, H, W, 3)); v_a = rng.normal(size=(C, H, W))
        p = oracle.project(sc, o)
        _, ids0, offs0 = oracle.isect(p, C, N, W, H, o)
        b = oracle.render_bwd(p, C, N, W, H, o, v_img, v_a)
        g = oracle.project_bwd(sc, p, b["v2d"], o)
        grads = {"means": g["v_means"], "quats": g["v_quats"], "scales": g["v_scales"],
                 "opacities": g["v_opacities"], "colors": g["v_colors"]}
        vis_any = (p["radii"][..., 0] > 0).any(axis=0)
        checked = 0
        worst = 0.0
        for name, G in grads.items():
            flatG = G.reshape(N, -1)
            for n in np.nonzero(vis_any)[0][:10]:
                for j in range(flatG.shape[1]):
                    if name == "colors" and j >= 3 * (sh + 1) ** 2:
                        continue
                    x0 = sc[name].reshape(N, -1)[n, j]
                    h = np.float32(1e-6 * max(1.0, abs(float(x0))))
                    vals = []
                    steps = []
                    for sgn in (+1, -1):
                        sc2 = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in sc.items()}
                        arr = sc2[name].reshape(N, -1)
                        arr[n, j] = np.float32(x0 + sgn * h)
                        steps.append(float(arr[n, j]) - float(x0))
                        l, (ids1, offs1) = _loss(sc2, o, v_img, v_a)
                        if not (np.array_equal(ids1, ids0) and np.array_equal(offs1, offs0)):
                            vals = None
                            break
                        vals.append(l)
                    if vals is None:
                        continue
                    fd = (vals[0] - vals[1]) / (steps[0] - steps[1])
                    an = flatG[n, j]
                    err = abs(an - fd) / max(abs(fd), 1e-4)
                    worst = max(worst, err)
                    assert abs(an - fd) <= 2e-4 * abs(fd) + 1e-6, (name, n, j, an, fd)
                    checked += 1
        assert checked > 80, checked

    @pytest.mark.parametrize("seed,sh", [(0, 0), (1, 2)])
    def test_clamped_J_gradient_matches_fd(self, oracle_lib, seed, sh):
        """Q27 gradient branch (the clamped coordinate gets no gradient
        through J, and t_z enters J through t_c = t_z u_c): splats deep inside the clamp
        (|t_x/t_z| 1.1-1.5 against a 0.65 limit) whose 3-sigma boxes still reach the image;
        every parameter gradient of those splats = central FD over the fp32 inputs."""
        o = oracle.Options(sh_degree=sh, amb_rel_floor=2e-3)
        W = H = 32
        found = None
        for k in range(300):
            sc = S.tiny_scene(seed * 1000 + 500 + k, N=20, width=W, height=H, sh_degree=sh)
            rng = np.random.default_rng(seed * 1000 + k)
            m = 4
            z = rng.uniform(1.2, 2.0, m)
            u = rng.choice([-1, 1], m) * rng.uniform(1.1, 1.5, m)
            v = rng.uniform(-0.3, 0.3, m)
            sc["means"][:m] = np.stack([u * z, v * z, z], 1)
            sc["scales"][:m] = rng.uniform(0.35, 0.6, (m, 3))
            sc["opacities"][:m] = rng.uniform(0.3, 0.8, m)
            p = oracle.project(sc, o)
            r = oracle.render_fwd(p, 1, 20, W, H, o)
            vis = p["radii"][0, :m, 0] > 0
            if vis.sum() >= 2 and not r["ambig"].any():
                found = (sc, np.nonzero(vis)[0])
                break
        assert found is not None
        sc, clamped = found
        N = sc["means"].shape[0]
        rng = np.random.default_rng(seed)
        v_img = rng.normal(size=(1, H, W, 3)); v_a = rng.normal(size=(1, H, W))
        p = oracle.project(sc, o)
        _, ids0, offs0 = oracle.isect(p, 1, N, W, H, o)
        b = oracle.render_bwd(p, 1, N, W, H, o, v_img, v_a)
        g = oracle.project_bwd(sc, p, b["v2d"], o)
        grads = {"means": g["v_means"], "quats": g["v_quats"], "scales": g["v_scales"],
                 "opacities": g["v_opacities"]}
        checked = 0
        for name, G in grads.items():
            flatG = G.reshape(N, -1)
            for n in clamped:
                for j in range(flatG.shape[1]):
                    x0 = sc[name].reshape(N, -1)[n, j]
                    h = np.float32(1e-5 * max(1.0, abs(float(x0))))
                    vals, steps = [], []
                    for sgn in (+1, -1):
                        sc2 = {kk: (vv.copy() if isinstance(vv, np.ndarray) else vv) for kk, vv in sc.items()}
                        arr = sc2[name].reshape(N, -1)
                        arr[n, j] = np.float32(x0 + sgn * h)
                        steps.append(float(arr[n, j]) - float(x0))
                        l, (ids1, offs1) = _loss(sc2, o, v_img, v_a)
                        if not (np.array_equal(ids1, ids0) and np.array_equal(offs1, offs0)):
                            vals = None
                            break
                        vals.append(l)
                    if vals is None:
                        continue
                    fd = (vals[0] - vals[1]) / (steps[0] - steps[1])
                    an = flatG[n, j]
                    assert abs(an - fd) <= 2e-4 * abs(fd) + 1e-6, (name, n, j, an, fd)
                    checked += 1
        assert checked >= 16, checked

    def test_projection_backward_bound_dominates(self, oracle_lib):
        """The absmode tolerance model is |Jacobian| e: for any perturbation d of the 2D
        gradients, |project_bwd(v + d) - project_bwd(v)| <= project_bwd_bound(|d|), and
        |project_bwd(v)| <= project_bwd_bound(|v|) (triangle inequality, linearity)."""
        for sh, aa in [(0, 0), (3, 1)]:
            sc = S.tiny_scene(31 + sh, N=80, width=48, height=40, sh_degree=sh, views=2)
            o = oracle.Options(sh_degree=sh, antialiased=aa)
            p = oracle.project(sc, o)
            rng = np.random.default_rng(sh)
            v = rng.normal(size=(2, 80, 9)); d = rng.normal(size=(2, 80, 9)) * 1e-3
            vz = rng.normal(size=(2, 80)); dz = rng.normal(size=(2, 80)) * 1e-3
            g0 = oracle.project_bwd(sc, p, v, o, vz=vz, pose=True)
            g1 = oracle.project_bwd(sc, p, v + d, o, vz=vz + dz, pose=True)
            bd = oracle.project_bwd_bound(sc, p, d, o, ez=dz, pose=True)
            bv = oracle.project_bwd_bound(sc, p, v, o, ez=vz, pose=True)
            for k in g0:
                assert np.all(np.abs(g1[k] - g0[k]) <= bd[k] * (1 + 1e-9) + 1e-300), k
                assert np.all(np.abs(g0[k]) <= bv[k] * (1 + 1e-9) + 1e-300), k
                assert bv[k].max() > 0

    def test_dp_linearity(self, oracle_lib):
        """Q30 / 8(e): gradients of two views = sum of per-view gradients (sharding invariant)."""
        sc, o = _clean_scene(7, sh_degree=1, views=2)
        C, N, W, H = 2, sc["means"].shape[0], sc["width"], sc["height"]
        rng = np.random.default_rng(7)
        v_img = rng.normal(size=(C, H, W, 3))
        res = oracle.forward_backward(sc, o, v_img, with_isect=False)
        tot = None
        for c in range(C):
            s1 = dict(sc); s1["viewmats"] = sc["viewmats"][c:c + 1]; s1["Ks"] = sc["Ks"][c:c + 1]
            r1 = oracle.forward_backward(s1, o, v_img[c:c + 1], with_isect=False)["grads"]
            tot = r1 if tot is None else {k: tot[k] + r1[k] for k in tot}
        for k in tot:
            assert np.allclose(tot[k], res["grads"][k], rtol=1e-12, atol=1e-15)


class TestPacked:
    """Q29: packed items are the visible (c,n) pairs, camera-major then by n."""

    def test_pack_order_bruteforce(self, oracle_lib):
        rng = np.random.default_rng(5)
        C, N = 3, 50
        radii = rng.integers(0, 3, size=(C, N, 2)).astype(np.int32)
        cam, gid, index = oracle.pack(dict(radii=radii))
        exp = [(c, n) for c in range(C) for n in range(N) if radii[c, n, 0] > 0 and radii[c, n, 1] > 0]
        assert list(zip(cam.tolist(), gid.tolist())) == exp
        for i, (c, n) in enumerate(exp):
            assert index[c, n] == i
        assert (index >= 0).sum() == len(exp)

    def test_packed_keys_are_dense_keys(self, oracle_lib):
        """Tile keys do not depend on the storage layout; the values re-index through
        pack()'s map (SURVEY 8c 'Dense vs packed')."""
        sc = S.tiny_scene(3, N=300, width=96, height=80, sh_degree=0, views=2)
        o = oracle.Options(sh_degree=0)
        p = oracle.project(sc, o)
        C, N = 2, 300
        keys, ids, offs = oracle.isect(p, C, N, 96, 80, o)
        cam, gid, index = oracle.pack(p)
        assert np.all(index.reshape(-1)[ids] >= 0)          # every intersected item is packed
        packed_ids = index.reshape(-1)[ids]
        assert np.array_equal(cam[packed_ids] * N + gid[packed_ids], ids)



# --------------------------------------------------------------------------- depth rendering, pose gradients
class TestDepthAndPose:
    """NEXT-2 (accumulated / expected depth) and NEXT-3 (camera pose gradients,
    P:233-239) in the oracle: closed forms and central finite differences."""

    def test_depth_closed_forms(self, oracle_lib):
        o = oracle.Options()
        # one splat: alpha at the centre = o_eff; expected depth = its depth for any alpha
        p = _splat2d([[5.5, 5.5]], [[1, 0, 1]], [0.3], [[0.3, 0.4, 0.5]], [2.5], [[3, 3]])
        r = oracle.render_fwd(p, 1, 1, 16, 16, o)
        assert r["depth"][0, 5, 5] == pytest.approx(0.3 * 2.5, rel=1e-7)
        assert r["depth_exp"][0, 5, 5] == pytest.approx(2.5, rel=1e-6)
        assert r["depth"][0, 0, 0] == 0 and r["depth_exp"][0, 0, 0] == 0   # nothing composited
        # two splats, alpha 0.5 each, depths 1 then 2: acc = 0.5*1 + 0.25*2, exp = acc / 0.75
        p = _splat2d([[5.5, 5.5], [5.5, 5.5]], [[1, 0, 1], [1, 0, 1]], [0.5, 0.5], [[1, 0, 0], [0, 1, 0]],
                     [1.0, 2.0], [[3, 3], [3, 3]])
        r = oracle.render_fwd(p, 1, 2, 16, 16, o)
        assert r["depth"][0, 5, 5] == pytest.approx(1.0, rel=1e-7)
        assert r["depth_exp"][0, 5, 5] == pytest.approx(1.0 / 0.75, rel=1e-7)

    @pytest.mark.parametrize("seed", [0, 1])
    def test_depth_render_bwd_matches_fd(self, oracle_lib, seed):
        """dL/d(mean2d, conic, opac_eff, depth) for L = <v_C, C> + <v_D, D_acc> + <v_E, D_exp>
        equals central FD of the f64 render."""
        sc, o = _clean_scene(seed + 40, sh_degree=0)
        C, N, W, H = 1, sc["means"].shape[0], sc["width"], sc["height"]
        p = oracle.project(sc, o)
        rng = np.random.default_rng(seed)
        v_img = rng.normal(size=(C, H, W, 3)); v_d = rng.normal(size=(C, H, W)); v_e = rng.normal(size=(C, H, W))
        b = oracle.render_bwd(p, C, N, W, H, o, v_img, v_depth=v_d, v_depth_exp=v_e)

        def L(pp):
            r = oracle.render_fwd(pp, C, N, W, H, o)
            return (r["rgb"] * v_img).sum() + (r["depth"] * v_d).sum() + (r["depth_exp"] * v_e).sum()
        fields = [("mean2d", 0, 2), ("conic", 2, 3), ("opac_eff", 8, 1), ("depth", None, 1)]
        checked = 0
        for n in np.nonzero(p["radii"][0, :, 0] > 0)[0]:
            for name, off, k in fields:
                for j in range(k):
                    h = 1e-6
                    pp = {kk: vv.copy() for kk, vv in p.items()}
                    arr = pp[name].reshape(C, N, -1)
                    arr[0, n, j] += h; lp = L(pp)
                    arr[0, n, j] -= 2 * h; lm = L(pp)
                    fd = (lp - lm) / (2 * h)
                    an = b["vz"][0, n] if off is None else b["v2d"][0, n, off + j]
                    assert abs(an - fd) <= 1e-5 * abs(fd) + 1e-6, (name, n, j, an, fd)
                    checked += 1
        assert checked > 40

    @pytest.mark.parametrize("seed,sh", [(0, 0), (1, 3)])
    def test_depth_full_chain_and_pose_match_fd(self, oracle_lib, seed, sh):
        """Through the projection: dL/d means (incl. the depth = t_z path) and dL/d viewmats
        (t, Sigma_c and SH view-direction paths) equal central FD over the f32 inputs."""
        sc, o = _clean_scene(seed + 60, sh_degree=sh, views=2)
        C, N, W, H = 2, sc["means"].shape[0], sc["width"], sc["height"]
        rng = np.random.default_rng(seed)
        v_img = rng.normal(size=(C, H, W, 3)); v_a = rng.normal(size=(C, H, W))
        v_d = rng.normal(size=(C, H, W)); v_e = rng.normal(size=(C, H, W))
        p = oracle.project(sc, o)
        _, ids0, offs0 = oracle.isect(p, C, N, W, H, o)
        b = oracle.render_bwd(p, C, N, W, H, o, v_img, v_a, v_depth=v_d, v_depth_exp=v_e)
        g = oracle.project_bwd(sc, p, b["v2d"], o, vz=b["vz"], pose=True)

        def fd_of(name, idx):
            x0 = sc[name].reshape(-1)[idx]
            h = np.float32(1e-6 * max(1.0, abs(float(x0))))
            vals, steps = [], []
            for sgn in (+1, -1):
                sc2 = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in sc.items()}
                arr = sc2[name].reshape(-1)
                arr[idx] = np.float32(x0 + sgn * h)
                steps.append(float(arr[idx]) - float(x0))
                l, (ids1, offs1) = _loss(sc2, o, v_img, v_a, v_d=v_d, v_e=v_e)
                if not (np.array_equal(ids1, ids0) and np.array_equal(offs1, offs0)):
                    return None
                vals.append(l)
            return (vals[0] - vals[1]) / (steps[0] - steps[1])
        checked = 0
        vis = np.nonzero((p["radii"][..., 0] > 0).any(axis=0))[0][:8]
        for n in vis:
            for j in range(3):
                fd = fd_of("means", 3 * n + j)
                if fd is None:
                    continue
                an = g["v_means"][n, j]
                assert abs(an - fd) <= 2e-4 * abs(fd) + 1e-6, ("means", n, j, an, fd)
                checked += 1
        for c in range(C):
            for i in range(3):
                for j in range(4):
                    fd = fd_of("viewmats", 16 * c + 4 * i + j)
                    if fd is None:
                        continue
                    an = g["v_viewmats"][c, i, j]
                    assert abs(an - fd) <= 2e-4 * abs(fd) + 1e-5 * (1 + abs(an)), ("viewmat", c, i, j, an, fd)
                    checked += 1
            assert np.all(g["v_viewmats"][c, 3] == 0)
        assert checked > 30, checked

    def test_pose_translation_identity(self, oracle_lib):
        """A.2: dL/dt (camera translation) = sum_n dL/d(camera-space mean) when the
        view direction does not enter (direct colours) and Sigma_c does not depend on w."""
        sc, o = _clean_scene(77, sh_degree=0, views=1)
        C, N, W, H = 1, sc["means"].shape[0], sc["width"], sc["height"]
        rng = np.random.default_rng(1)
        v_img = rng.normal(size=(C, H, W, 3))
        p = oracle.project(sc, o)
        b = oracle.render_bwd(p, C, N, W, H, o, v_img)
        g = oracle.project_bwd(sc, p, b["v2d"], o, pose=True)
        # with W = the view rotation, dL/dw = sum_n v_t(n) and dL/dmu_n = W^T v_t(n) (SH0: no
        # direction dependence), so dL/dw = W (sum_n dL/dmu_n)
        Wr = sc["viewmats"][0, :3, :3].astype(np.float64)
        np.testing.assert_allclose(g["v_viewmats"][0, :3, 3], Wr @ g["v_means"].sum(0), rtol=1e-9, atol=1e-12)


class TestNDFeatures:
    """N-dimensional rasterization: D-channel features composited like RGB."""

    def test_two_splats_closed_form(self, oracle_lib):
        o = oracle.Options()
        f = np.array([[1.0, 2.0, -1.0, 0.5, 3.0], [0.0, 4.0, 1.0, -2.0, 1.0]])
        p = _splat2d([[5.5, 5.5], [5.5, 5.5]], [[1, 0, 1], [1, 0, 1]], [0.5, 0.5], [[1, 0, 0], [0, 1, 0]],
                     [1.0, 2.0], [[3, 3], [3, 3]])
        r = oracle.render_fwd_nd(p, f, 1, 2, 16, 16, o)
        np.testing.assert_allclose(r["feat"][0, 5, 5], 0.5 * f[0] + 0.25 * f[1], rtol=1e-12)
        assert r["feat"][0, 0, 0].tolist() == [0.0] * 5

    def test_rgb_special_case_and_channel_independence(self, oracle_lib):
        """D = 3 features equal to the direct colours reproduce the RGB path; rendering D
        channels equals rendering any split of them (compositing is per channel)."""
        sc = S.tiny_scene(4, N=200, width=48, height=40, sh_degree=-1, views=2)
        o = oracle.Options(sh_degree=-1)
        p = oracle.project(sc, o)
        C, N = 2, 200
        rgb = oracle.render_fwd(p, C, N, 48, 40, o)
        nd = oracle.render_fwd_nd(p, sc["colors"], C, N, 48, 40, o)
        np.testing.assert_array_equal(nd["feat"], rgb["rgb"])
        np.testing.assert_array_equal(nd["T"], rgb["T"])
        f = np.random.default_rng(0).normal(size=(N, 7))
        full = oracle.render_fwd_nd(p, f, C, N, 48, 40, o)["feat"]
        a = oracle.render_fwd_nd(p, f[:, :2], C, N, 48, 40, o)["feat"]
        b = oracle.render_fwd_nd(p, f[:, 2:], C, N, 48, 40, o)["feat"]
        np.testing.assert_array_equal(full, np.concatenate([a, b], axis=-1))

    def test_nd_backward_matches_fd(self, oracle_lib):
        sc, o = _clean_scene(90, sh_degree=0)
        C, N, W, H = 1, sc["means"].shape[0], sc["width"], sc["height"]
        p = oracle.project(sc, o)
        rng = np.random.default_rng(3)
        D = 6
        f = rng.normal(size=(N, D))
        v = rng.normal(size=(C, H, W, D))
        va = rng.normal(size=(C, H, W))
        bg = rng.uniform(size=(C, D))
        b = oracle.render_bwd_nd(p, f, C, N, W, H, o, v, va, backgrounds=bg)

        def L(pp, ff):
            r = oracle.render_fwd_nd(pp, ff, C, N, W, H, o, backgrounds=bg)
            return (r["feat"] * v).sum() + (r["alpha"] * va).sum()
        checked = 0
        for n in np.nonzero(p["radii"][0, :, 0] > 0)[0][:10]:
            for j in range(D):
                h = 1e-6
                f2 = f.copy(); f2[n, j] += h; lp = L(p, f2)
                f2[n, j] -= 2 * h; lm = L(p, f2)
                fd = (lp - lm) / (2 * h)
                assert abs(b["v_colors"][n, j] - fd) <= 1e-6 * (1 + abs(fd)), (n, j)
                checked += 1
            for name, off, k in [("mean2d", 0, 2), ("conic", 2, 3), ("opac_eff", 8, 1)]:
                for j in range(k):
                    h = 1e-6
                    pp = {kk: vv.copy() for kk, vv in p.items()}
                    arr = pp[name].reshape(C, N, -1)
                    arr[0, n, j] += h; lp = L(pp, f)
                    arr[0, n, j] -= 2 * h; lm = L(pp, f)
                    fd = (lp - lm) / (2 * h)
                    an = b["v2d"][0, n, off + j]
                    assert abs(an - fd) <= 1e-5 * abs(fd) + 1e-7 * (1 + b["a2d"][0, n, off + j]), (name, n, j, an, fd)
                    checked += 1
        assert checked > 60


# --------------------------------------------------------------------------- Q36 (NEXT-4(ii))
class TestOpacityAwareExtent:
    """bbox_mode 2: the per-axis extent min(3, k) sigma with k^2 >= 2 ln(o_eff / alpha_min)
    (R1: alpha = o_eff exp(-sigma) >= alpha_min iff sigma <= ln(o_eff / alpha_min)).  Pinned by
    the closed form of the alpha support for isotropic splats and by output invariance: the
    method's images, transmittance, last splats and gradients are those of the 3-sigma box."""

    def test_isotropic_extent_brackets_the_alpha_support(self, oracle_lib):
        z, f = 2.0, 100.0
        for s in [0.01, 0.05, 0.2]:
            for op in [0.005, 0.02, 0.1, 0.3, 0.6, 0.99]:
                sc = _one_gaussian([0, 0, z], [1, 0, 0, 0], [s, s, s], op, [1, 1, 1],
                                   K=[[f, 0, 32], [0, f, 32], [0, 0, 1]])
                p0 = oracle.project(sc, oracle.Options(sh_degree=-1, fov_clamp=0, bbox_mode=0))
                p2 = oracle.project(sc, oracle.Options(sh_degree=-1, fov_clamp=0, bbox_mode=2))
                sig = math.sqrt(float(np.float32(s)) ** 2 * f * f / (z * z) + 0.3)   # S:129 closed form
                r0, r2 = p0["radii"][0, 0], p2["radii"][0, 0]
                assert r0.tolist() == [math.ceil(3 * sig)] * 2
                o32 = float(np.float32(op))
                if o32 < 1 / 255:
                    assert r2.tolist() == [0, 0]          # alpha < alpha_min everywhere: culled
                    continue
                k_true = math.sqrt(2 * math.log(o32 * 255))
                assert np.all(r2 <= r0)
                assert np.all(r2 >= min(3.0, k_true) * sig - 1e-6)             # contains the support
                assert np.all(r2 <= math.ceil(min(3.0, k_true * 1.02 + 0.1) * sig))   # and is tight
        # low opacity really shrinks the box (o = 0.02: k = sqrt(2 ln 5.1) = 1.81 vs 3)
        sc = _one_gaussian([0, 0, z], [1, 0, 0, 0], [0.2] * 3, 0.02, [1, 1, 1], K=[[f, 0, 32], [0, f, 32], [0, 0, 1]])
        r2 = oracle.project(sc, oracle.Options(sh_degree=-1, fov_clamp=0, bbox_mode=2))["radii"][0, 0]
        assert r2[0] <= 0.65 * math.ceil(3 * math.sqrt(0.04 * 2500 + 0.3))

    @pytest.mark.parametrize("name,aa", [("tiny", 0), ("tiny_sh3", 1), ("mip", 0), ("mip", 1), ("fig1", 0)])
    def test_output_invariance(self, oracle_lib, name, aa):
        if name == "tiny":
            sc = S.tiny_scene(3, N=300, sh_degree=0)
        elif name == "tiny_sh3":
            sc = S.tiny_scene(4, N=400, width=97, height=61, sh_degree=3, views=2)
        elif name == "mip":
            sc = S.mipnerf_like_scene(3000, width=96, height=64, views=1, sh_degree=1, seed=5)
        else:
            sc = S.fig1_scene()
        C, N, W, H = sc["viewmats"].shape[0], sc["means"].shape[0], sc["width"], sc["height"]
        v_img = np.random.default_rng(1).normal(size=(C, H, W, 3))
        res = {}
        for mode in (0, 2):
            o = oracle.Options(sh_degree=sc["sh_degree"], antialiased=aa, bbox_mode=mode)
            res[mode] = oracle.forward_backward(sc, o, v_img)
            res[mode]["M"] = res[mode]["keys"].size
        a, b = res[0], res[2]
        assert b["M"] <= a["M"]
        for k in ("rgb", "alpha", "T", "last_gid"):
            assert np.array_equal(a["fwd"][k], b["fwd"][k]), k
        for k, g in a["grads"].items():
            assert np.array_equal(g, b["grads"][k]), k
        if name == "mip":
            assert b["M"] < a["M"]


# --------------------------------------------------------------------------- NEXT-1
class TestDensificationStats:
    """Absgrad (App. Absgrad) and the ADC statistics."""

    def test_absgrad_equals_sum_of_single_pixel_gradients(self, oracle_lib):
        """Brute force: the per-pixel absolute view-space gradient sums equal the sum over
        pixels p of |v_mean2d| of the loss that keeps only pixel p (linearity of B1-B6 in v_C)."""
        sc = S.tiny_scene(6, N=40, width=20, height=18, sh_degree=0)
        o = oracle.Options(sh_degree=0)
        p = oracle.project(sc, o)
        v_img = np.random.default_rng(2).normal(size=(1, 18, 20, 3))
        full = oracle.render_bwd(p, 1, 40, 20, 18, o, v_img)
        acc = np.zeros((1, 40, 2))
        for y in range(18):
            for x in range(20):
                vp = np.zeros_like(v_img)
                vp[0, y, x] = v_img[0, y, x]
                acc += np.abs(oracle.render_bwd(p, 1, 40, 20, 18, o, vp)["v2d"][..., 0:2])
        assert np.allclose(full["absgrad"], acc, rtol=1e-12, atol=1e-18)
        assert np.all(full["absgrad"] >= np.abs(full["v2d"][..., 0:2]) - 1e-15)
        assert (full["absgrad"] > np.abs(full["v2d"][..., 0:2]) * (1 + 1e-9)).any()   # cancellation exists

    def test_stats_special_cases(self, oracle_lib):
        rng = np.random.default_rng(3)
        C, N = 4, 50
        radii = rng.integers(0, 9, size=(C, N, 2)).astype(np.int32)
        radii[rng.uniform(size=(C, N)) < 0.3] = 0
        g = rng.normal(size=(C, N, 2))
        st = oracle.densify_stats(radii, g)
        vis = (radii[..., 0] > 0) & (radii[..., 1] > 0)
        # one camera: the norm of that view's gradient (library routine)
        one = oracle.densify_stats(radii[:1], g[:1])
        assert np.allclose(one["grad2d"], np.where(vis[0], np.linalg.norm(g[0], axis=-1), 0))
        # camera order does not matter; counts are the visible views; homogeneity in the scale
        perm = oracle.densify_stats(radii[::-1], g[::-1])
        assert np.allclose(perm["grad2d"], st["grad2d"]) and np.array_equal(perm["count"], st["count"])
        assert np.array_equal(st["count"], vis.sum(0))
        sc2 = oracle.densify_stats(radii, g, scale=(2.0, 2.0), radius_scale=0.5)
        assert np.allclose(sc2["grad2d"], 2 * st["grad2d"]) and np.allclose(sc2["max_radii"], 0.5 * st["max_radii"])
        # invisible everywhere -> zeros
        none = oracle.densify_stats(np.zeros_like(radii), g)
        assert not none["grad2d"].any() and not none["count"].any() and not none["max_radii"].any()
