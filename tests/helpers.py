"""Test helpers: tiny hand-built scenes (data only — no method arithmetic)."""
import numpy as np

import scenegen as sg


def one_gaussian(mean, scales, quat=(1.0, 0.0, 0.0, 0.0), opacity=0.8, dc=(0.3, -0.2, 0.1), rest=None):
    K = 16
    sh = np.zeros((K, 3, 1))
    sh[0, :, 0] = dc
    if rest is not None:
        sh[1:, :, 0] = np.asarray(rest).reshape(15, 3)
    return sg.make_scene(np.asarray(mean, float).reshape(3, 1), np.asarray(scales, float).reshape(3, 1),
                         np.asarray(quat, float).reshape(4, 1), [opacity], sh)


def concat(*scenes):
    return sg.make_scene(np.concatenate([s.means for s in scenes], 1), np.concatenate([s.scales for s in scenes], 1),
                         np.concatenate([s.rotations for s in scenes], 1),
                         np.concatenate([s.opacities for s in scenes]), np.concatenate([s.sh for s in scenes], 2))


def quat_to_rot_scipy(q_wxyz):
    from scipy.spatial.transform import Rotation
    w, x, y, z = q_wxyz
    return Rotation.from_quat([x, y, z, w]).as_matrix()


def random_cam(rng, width=64, height=48, f=60.0):
    eye = rng.normal(size=3)
    eye = eye / np.linalg.norm(eye) * rng.uniform(3.0, 5.0)
    R, t = sg.look_at(eye, rng.normal(scale=0.2, size=3))
    return sg.Camera(f, f * rng.uniform(0.9, 1.1), width / 2 + rng.uniform(-3, 3), height / 2 + rng.uniform(-3, 3),
                     width, height, R, t, 0.2)


def dense_scene(seed, n, width=64, height=64, f=64.0, zr=(2.0, 6.0), smin=0.02, smax=0.3):
    """n Gaussians in the frustum of camera_identity(width, height, f): a denser C0."""
    rng = np.random.default_rng(seed)
    z = rng.uniform(*zr, n)
    x = rng.uniform(-0.55, 0.55, n) * z * width / f
    y = rng.uniform(-0.55, 0.55, n) * z * height / f
    s = np.exp(rng.uniform(np.log(smin), np.log(smax), (3, n)))
    fl = rng.random(n) < 0.3
    s[2, fl] *= np.exp(rng.uniform(np.log(1e-2), 0, fl.sum()))
    return sg.make_scene(np.stack([x, y, z]), s, sg.random_quaternions(rng, n), sg.opacity_mixture(rng, n),
                         sg.sh_coeffs(rng, n))
