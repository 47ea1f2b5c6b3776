"""Seeded synthetic inputs standing in for the paper's datasets.

The reference is measured on ICL-NUIM / TUM RGB-D, which
are not available here; BASELINE.json's configs C1-C5 describe the
replacement: random Perlin-textured planes (and boxes for C3), pinhole
intrinsics, tracked-frame poses 2-10 cm / <=2 deg from the keyframe, and CNN
priors = ground truth + noise with per-pixel uncertainty. SURVEY.md 8(d)
fixes the remaining details; this module implements them with numpy's PCG64
generator (seed per (scene, frame) derived with the reference's mix_seed,
pipeline.hpp:87-92).

Also restates the reference's analytic test fixture PlaneScene /
render_view (tests/support/synthetic.hpp:25-72), used by the KAT tests.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from ._ffi import CameraIntrinsics, PredictionSet, SearchConfig

MASK64 = (1 << 64) - 1


def mix_seed(seed: int, salt: int) -> int:
    """pipeline.hpp:87-92 (splitmix64 finaliser)."""
    z = (seed + (salt + 1) * 0x9E3779B97F4A7C15) & MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


# --------------------------------------------------------------------------
# quaternion helpers (w, x, y, z)
def quat_to_matrix(q) -> np.ndarray:
    w, x, y, z = q
    tx, ty, tz = 2 * x, 2 * y, 2 * z
    twx, twy, twz = tx * w, ty * w, tz * w
    txx, txy, txz = tx * x, ty * x, tz * x
    tyy, tyz, tzz = ty * y, tz * y, tz * z
    return np.array([[1 - (tyy + tzz), txy - twz, txz + twy],
                     [txy + twz, 1 - (txx + tzz), tyz - twx],
                     [txz - twy, tyz + twx, 1 - (txx + tyy)]])


def axis_angle_quat(axis, angle) -> np.ndarray:
    axis = np.asarray(axis, float)
    axis = axis / np.linalg.norm(axis)
    s = math.sin(angle / 2)
    return np.array([math.cos(angle / 2), axis[0] * s, axis[1] * s, axis[2] * s])


IDENTITY_Q = np.array([1.0, 0.0, 0.0, 0.0])
ENV_GAIN, ENV_BIAS = 4.0, 0.1


# --------------------------------------------------------------------------
# Perlin gradient noise (Perlin 2002, "improved noise", 2-D), seeded
class Perlin2D:
    def __init__(self, rng: np.random.Generator):
        p = rng.permutation(256)
        self.perm = np.concatenate([p, p]).astype(np.int64)
        ang = rng.uniform(0, 2 * np.pi, 256)
        self.gx, self.gy = np.cos(ang), np.sin(ang)

    @staticmethod
    def _fade(t):
        return t * t * t * (t * (t * 6 - 15) + 10)

    def noise(self, x, y):
        xi = np.floor(x).astype(np.int64)
        yi = np.floor(y).astype(np.int64)
        xf, yf = x - xi, y - yi
        xi &= 255
        yi &= 255
        perm = self.perm

        def grad(ix, iy, dx, dy):
            h = perm[perm[ix] + iy]
            return self.gx[h] * dx + self.gy[h] * dy

        n00 = grad(xi, yi, xf, yf)
        n10 = grad(xi + 1, yi, xf - 1, yf)
        n01 = grad(xi, yi + 1, xf, yf - 1)
        n11 = grad(xi + 1, yi + 1, xf - 1, yf - 1)
        u, v = self._fade(xf), self._fade(yf)
        return (n00 * (1 - u) + n10 * u) * (1 - v) + (n01 * (1 - u) + n11 * u) * v

    def fbm(self, x, y, octaves=4, lacunarity=2.0, gain=0.5):
        s = np.zeros_like(x)
        amp, freq, norm = 1.0, 1.0, 0.0
        for _ in range(octaves):
            s += amp * self.noise(x * freq, y * freq)
            norm += amp
            amp *= gain
            freq *= lacunarity
        return s / norm


# --------------------------------------------------------------------------
@dataclass
class Plane:
    normal: np.ndarray  # unit, world
    offset: float       # n . X = offset
    origin: np.ndarray  # point on the plane (texture origin)
    e1: np.ndarray
    e2: np.ndarray
    noise: Perlin2D
    freq: float
    flat: Perlin2D | None = None  # textureless-region field (C5)
    # box faces are bounded: |(X-origin).e1| <= half1, |(X-origin).e2| <= half2
    half1: float = math.inf
    half2: float = math.inf


@dataclass
class ConfigSpec:
    name: str
    width: int
    height: int
    fx: float
    fy: float
    cx: float
    cy: float
    frames: int
    planes: tuple = (3, 3)
    boxes: bool = False
    depth_range: tuple = (0.5, 4.0)
    normal_max_deg: float = 40.0
    trans_range: tuple = (0.02, 0.10)
    rot_max_deg: float = 2.0
    pixel_noise: float = 0.01
    logsigma_range: tuple = (-3.0, -1.0)
    grad_sigma: float = 0.05
    textureless_frac: float = 0.0
    laplace_b: float | None = None
    search: SearchConfig = field(default_factory=SearchConfig)
    gn_iterations: int = 10
    keyframes: int = 1

    def camera(self) -> CameraIntrinsics:
        return CameraIntrinsics(self.fx, self.fy, self.cx, self.cy, self.width, self.height)


# BASELINE.json configs
CONFIGS = {
    "C1": ConfigSpec("C1", 320, 240, 262.5, 262.5, 160.0, 120.0, frames=5, gn_iterations=50),
    "C2": ConfigSpec("C2", 640, 480, 525.0, 525.0, 320.0, 240.0, frames=10),
    "C3": ConfigSpec("C3", 640, 480, 525.0, 525.0, 320.0, 240.0, frames=10, planes=(3, 8),
                     boxes=True, keyframes=64),
    "C4": ConfigSpec("C4", 3840, 2160, 3000.0, 3000.0, 1920.0, 1080.0, frames=8,
                     gn_iterations=500),
    "C5": ConfigSpec("C5", 640, 480, 525.0, 525.0, 320.0, 240.0, frames=20,
                     textureless_frac=0.3, laplace_b=0.2, search=SearchConfig(0.1, 20.0)),
}


def small_spec(width=96, height=72, frames=3, **kw) -> ConfigSpec:
    """A C2-like scene at test size (focal scaled with the width)."""
    f = 525.0 * width / 640.0
    return ConfigSpec(f"S{width}x{height}", width, height, f, f, width / 2.0, height / 2.0,
                      frames=frames, **kw)


def _unit(v):
    return v / np.linalg.norm(v)


def _random_normal(rng, max_deg):
    # direction within max_deg of -z (facing the camera), uniform in solid angle
    cmax = math.cos(math.radians(max_deg))
    c = rng.uniform(cmax, 1.0)
    phi = rng.uniform(0, 2 * math.pi)
    s = math.sqrt(max(0.0, 1 - c * c))
    return np.array([s * math.cos(phi), s * math.sin(phi), c])


def _basis(n):
    a = np.array([1.0, 0, 0]) if abs(n[0]) < 0.9 else np.array([0, 1.0, 0])
    e1 = _unit(np.cross(n, a))
    e2 = np.cross(n, e1)
    return e1, e2


@dataclass
class Scene:
    spec: ConfigSpec
    planes: list
    seed: int


def make_scene(spec: ConfigSpec, seed: int) -> Scene:
    """Random planes (and boxes): the deepest plane is unbounded (background),
    the nearer ones are rectangles covering part of the view, so every
    keyframe shows several depths and occlusion edges."""
    rng = np.random.default_rng(mix_seed(seed, 0))
    lo, hi = spec.planes
    n = int(rng.integers(lo, hi + 1))
    depths = np.sort(rng.uniform(*spec.depth_range, n))[::-1]  # far -> near
    planes = []
    tex_freq = 12.0  # detail cycles per metre; fBm adds 2 octaves above it
    tan_x = spec.width / (2 * spec.fx)
    tan_y = spec.height / (2 * spec.fy)
    for k in range(n):
        prng = np.random.default_rng(mix_seed(seed, 100 + k))
        d = float(depths[k])
        flat = None
        if spec.textureless_frac > 0:
            flat = Perlin2D(prng)
        freq = tex_freq * prng.uniform(0.7, 1.4)
        if k == 0 or not (spec.boxes and prng.uniform() < 0.5):
            nrm = _random_normal(prng, spec.normal_max_deg)
            # centre on the ray through a random point of the central view
            u = prng.uniform(-0.6, 0.6) * tan_x
            v = prng.uniform(-0.6, 0.6) * tan_y
            origin = np.array([u * d, v * d, d])
            e1, e2 = _basis(nrm)
            half = math.inf if k == 0 else float(prng.uniform(0.25, 0.6) * d * tan_x)
            planes.append(Plane(nrm, float(nrm @ origin), origin, e1, e2, Perlin2D(prng), freq,
                                flat, half, half))
        else:
            # box: its three camera-facing faces as bounded planes
            u = prng.uniform(-0.5, 0.5) * tan_x
            v = prng.uniform(-0.5, 0.5) * tan_y
            c = np.array([u * d, v * d, d])
            half = float(prng.uniform(0.1, 0.25) * d * tan_x)
            rot = quat_to_matrix(axis_angle_quat(prng.normal(size=3),
                                                 math.radians(prng.uniform(0, 35))))
            for ax in range(3):
                nrm = rot[:, ax].copy()
                if nrm[2] > 0:
                    nrm = -nrm  # the face looking at the camera
                origin = c + nrm * half
                e1, e2 = rot[:, (ax + 1) % 3].copy(), rot[:, (ax + 2) % 3].copy()
                planes.append(Plane(nrm, float(nrm @ origin), origin, e1, e2, Perlin2D(prng),
                                    freq, flat, half, half))
    return Scene(spec, planes, seed)


def render(scene: Scene, q, t, rng: np.random.Generator | None = None):
    """Render intensity (float32, [0,1]) and z-depth (float64) for camera pose
    T_WC = (q, t). Nearest positive ray/plane hit; Perlin texture in each
    plane's own coordinates (multi-view consistent); optional pixel noise."""
    spec = scene.spec
    h, w = spec.height, spec.width
    R = quat_to_matrix(q)
    ys, xs = np.mgrid[0:h, 0:w].astype(np.float64)
    dc = np.stack([(xs - spec.cx) / spec.fx, (ys - spec.cy) / spec.fy, np.ones_like(xs)], -1)
    dw = dc @ R.T
    o = np.asarray(t, float)
    best_t = np.full((h, w), np.inf)
    best_k = np.full((h, w), -1, np.int64)
    for k, pl in enumerate(scene.planes):
        den = dw @ pl.normal
        with np.errstate(divide="ignore", invalid="ignore"):
            th = (pl.offset - pl.normal @ o) / den
        ok = (th > 1e-6) & np.isfinite(th)
        if np.isfinite(pl.half1):
            X = o + th[..., None] * dw
            rel = X - pl.origin
            ok &= (np.abs(rel @ pl.e1) <= pl.half1) & (np.abs(rel @ pl.e2) <= pl.half2)
        upd = ok & (th < best_t)
        best_t[upd] = th[upd]
        best_k[upd] = k
    if np.any(best_k < 0):
        # background: far fronto-parallel wall (never reached for C1-C5 poses)
        miss = best_k < 0
        best_t[miss] = (spec.depth_range[1] * 3 - o[2]) / np.maximum(dw[..., 2][miss], 1e-3)
    X = o + best_t[..., None] * dw
    inten = np.full((h, w), 0.5)
    for k, pl in enumerate(scene.planes):
        sel = best_k == k
        if not np.any(sel):
            continue
        rel = X[sel] - pl.origin
        a, b = rel @ pl.e1, rel @ pl.e2
        # patchy texture like the reference fixture (synthetic.hpp:38-46): a
        # smooth base plus high-frequency detail gated by a low-frequency
        # envelope, so that roughly a third of the pixels pass the default
        # 0.02 texture threshold
        base = 0.5 + 0.3 * pl.noise.fbm(a * 2.0 + 0.37 * k, b * 2.0 + 0.71 * k, octaves=2)
        env = np.clip(ENV_GAIN * pl.noise.noise(a * 1.3 + 11.1, b * 1.3 + 7.7) + ENV_BIAS, 0, 1)
        high = pl.noise.fbm(a * pl.freq + 17.3 * k, b * pl.freq + 5.1 * k, octaves=3)
        v = base + env * 0.8 * high
        if pl.flat is not None:
            fl = pl.flat.noise(a * 2.0 + 3.7, b * 2.0 + 1.3)
            # constant-intensity regions covering ~textureless_frac of the area
            v = np.where(fl < _flat_threshold(spec.textureless_frac), 0.5, v)
        inten[sel] = v
    if rng is not None and spec.pixel_noise > 0:
        inten = inten + rng.normal(0.0, spec.pixel_noise, inten.shape)
    inten = np.clip(inten, 0.0, 1.0).astype(np.float32)
    depth = best_t  # dir_cam.z == 1 -> ray parameter == z-depth in the camera
    return inten, depth


def _flat_threshold(frac: float) -> float:
    # single-octave Perlin values are ~N(0, 0.2^2)-ish; the quantile map below
    # was fitted on 1e6 samples
    table = {0.1: -0.19, 0.2: -0.12, 0.3: -0.07, 0.4: -0.03, 0.5: 0.0}
    return table.get(round(frac, 1), -0.07)


def _q(v):
    return np.asarray(v, np.float64).astype(np.float32).astype(np.float64)


def make_predictions(spec: ConfigSpec, gt: np.ndarray, seed: int) -> PredictionSet:
    """CNN-prior stand-in: ln gt + N(0, sigma^2) with per-pixel
    ln sigma ~ U[-3,-1] (C5: Laplace(b) noise), gradients = forward
    differences of ln gt + N(0, 0.05^2); every value quantised through float
    like synth_oracle (predictions.hpp:201-203)."""
    rng = np.random.default_rng(mix_seed(seed, 7))
    h, w = gt.shape
    lg = np.log(gt)
    if spec.laplace_b is not None:
        noise = rng.laplace(0.0, spec.laplace_b, (h, w))
        var = np.full((h, w), 2.0 * spec.laplace_b ** 2)
    else:
        lsig = rng.uniform(*spec.logsigma_range, (h, w))
        sig = np.exp(lsig)
        noise = rng.normal(0.0, 1.0, (h, w)) * sig
        var = sig * sig
    log_depth = lg + noise
    gx = np.zeros((h, w))
    gy = np.zeros((h, w))
    gx[:, :-1] = lg[:, 1:] - lg[:, :-1] + rng.normal(0.0, spec.grad_sigma, (h, w - 1))
    gy[:-1, :] = lg[1:, :] - lg[:-1, :] + rng.normal(0.0, spec.grad_sigma, (h - 1, w))
    gv = np.full((h, w), spec.grad_sigma ** 2)
    return PredictionSet(_q(log_depth), _q(var), _q(gx), _q(gv), _q(gy), _q(gv),
                         source_focal=spec.fx)


@dataclass
class Sequence:
    spec: ConfigSpec
    I0: np.ndarray
    gt_depth: np.ndarray
    pred: PredictionSet
    frames: list  # list of (q_wxyz, t, I1)
    seed: int


def random_pose(spec: ConfigSpec, rng: np.random.Generator):
    d = rng.normal(size=3)
    d /= np.linalg.norm(d)
    t = d * rng.uniform(*spec.trans_range)
    ax = rng.normal(size=3)
    ang = math.radians(rng.uniform(0.0, spec.rot_max_deg))
    return axis_angle_quat(ax, ang), t


def make_sequence(spec: ConfigSpec, seed: int = 0, frames: int | None = None) -> Sequence:
    """Keyframe at the identity pose plus `frames` tracked frames."""
    scene = make_scene(spec, seed)
    I0, gt = render(scene, IDENTITY_Q, np.zeros(3), np.random.default_rng(mix_seed(seed, 1)))
    pred = make_predictions(spec, gt, seed)
    out = []
    nf = spec.frames if frames is None else frames
    for f in range(nf):
        rng = np.random.default_rng(mix_seed(seed, 1000 + f))
        q, t = random_pose(spec, rng)
        I1, _ = render(scene, q, t, rng)
        out.append((q, t, I1))
    return Sequence(spec, I0, gt, pred, out, seed)


# --------------------------------------------------------------------------
# The reference's analytic test fixture (tests/support/synthetic.hpp:25-72)
@dataclass
class PlaneScene:
    camera: CameraIntrinsics = field(
        default_factory=lambda: CameraIntrinsics(200.0, 200.0, 127.5, 95.5, 256, 192))
    z0: float = 2.0
    ax: float = 0.25
    ay: float = -0.15
    env_gain: float = 2.2
    env_bias: float = 0.5
    high_gain: float = 1.0

    def texture(self, u, v):
        base = 0.5 + 0.17 * np.sin(1.3 * u - 0.7 * v)
        s = np.sin(2.3 * u + 1.1 * v) * np.sin(1.7 * v - 0.9 * u + 0.4)
        env = np.clip(self.env_gain * s + self.env_bias, 0.0, 1.0)
        high = (0.13 * np.sin(31.0 * u + 7.0 * v) + 0.11 * np.sin(23.0 * u - 17.0 * v)
                + 0.08 * np.sin(43.0 * u + 29.0 * v))
        return np.clip(base + self.high_gain * env * high, 0.02, 0.98)


def render_view(scene: PlaneScene, q=IDENTITY_Q, t=(0.0, 0.0, 0.0)):
    """synthetic.hpp:54-72 -> (intensity float32, z-depth float64)"""
    K = scene.camera
    R = quat_to_matrix(q)
    o = np.asarray(t, float)
    n = np.array([-scene.ax, -scene.ay, 1.0])
    ys, xs = np.mgrid[0:K.height, 0:K.width].astype(np.float64)
    dc = np.stack([(xs - K.cx) / K.fx, (ys - K.cy) / K.fy, np.ones_like(xs)], -1)
    d = dc @ R.T
    th = (scene.z0 - n @ o) / (d @ n)
    P = o + th[..., None] * d
    return scene.texture(P[..., 0], P[..., 1]).astype(np.float32), th


def fronto_scene(focal: float) -> PlaneScene:
    """test_semidense.cpp:16-24"""
    return PlaneScene(CameraIntrinsics(focal, focal, 127.5, 95.5, 256, 192), ax=0.0, ay=0.0,
                      env_gain=10.0, env_bias=0.5)


def strong_pixel(img: np.ndarray):
    """test_semidense.cpp:33-47: strongest-gradient pixel away from borders."""
    v = img.astype(np.float32)
    h, w = v.shape
    best, out = -1.0, (64.0, 64.0)
    for y in range(20, h - 20):
        gx = 0.5 * (v[y, 21:w - 19] - v[y, 19:w - 21]).astype(np.float64)
        gy = 0.5 * (v[y + 1, 20:w - 20] - v[y - 1, 20:w - 20]).astype(np.float64)
        m = gx * gx + gy * gy
        k = int(np.argmax(m))
        if m[k] > best:
            best, out = float(m[k]), (float(20 + k), float(y))
    return out


def to_dfpred(pred: PredictionSet, source_focal: float) -> bytes:
    """The bytes save_predictions writes (predictions.hpp:125-145): 24-byte
    little-endian header {"DFPR", version 1, width, height, 6 channels,
    lround(focal * 1000)} and the six planes as float32 in channel order."""
    import struct
    h, w = pred.log_depth.shape
    focal_milli = int(math.floor(source_focal * 1000.0 + 0.5))  # std::lround for positives
    head = b"DFPR" + struct.pack("<5I", 1, w, h, 6, focal_milli)
    planes = [pred.log_depth, pred.log_depth_var, pred.grad_x, pred.grad_x_var, pred.grad_y,
              pred.grad_y_var]
    return head + b"".join(np.ascontiguousarray(p, dtype="<f4").tobytes() for p in planes)
