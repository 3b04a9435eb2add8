"""Seeded synthetic polar-Fourier workloads for the radial-SVD alignment path.

This module is HARNESS, not method: it produces the inputs (radial grid, template rings,
noisy rotated image rings) that both the CUDA path and the fp64 oracle consume.  It holds
none of the alignment arithmetic (no landscape, no kernel C, no basis, no compression).

Recipe (SURVEY.md §8(d) and gaps G11-G15, G19):

* Radial grid (§2.3): R Gauss-Jacobi(alpha=0, beta=1) nodes t_r on [-1,1]
  mapped by k = K (t+1)/2 with K = R-1 (reading G12), weights w_r = (K^2/4) omega_r so that
  sum_r g(k_r) w_r approximates int_0^K g(k) k dk.  Angular nodes psi_j = 2 pi j / Q.
* Molecule (G13): n_atoms isotropic Gaussian atoms, centres uniform in the ball of radius 0.3
  (units of the box half-width), sigma = 0.05, amplitude 1.
* Templates (G13/G14): central slices of the molecule's analytic 3-D Fourier transform,
  B(k, psi) = sum_a exp(-sigma^2 k^2 / 2) exp(-i k (cos psi e1 + sin psi e2) . c_a),
  for T view frames (e1, e2).  Tiny: uniform random views; otherwise a Fibonacci lattice.
* Images: image m is template t*(m) rotated in-plane by gamma_m ~ U[0, 2 pi) evaluated
  analytically off-grid, A_m(k, psi) = B_{t*}(k, psi - gamma_m), plus
  complex Gaussian noise with per-node variance sigma_hat^2 / (w_r dpsi),
  sigma_hat^2 = Pbar / (SNR R Q), Pbar = mean over images of sum_{r,j} w_r dpsi |signal|^2 (G11).
* Translations (G15/G19): each base image gets 9 copies multiplied by the phase ramp
  exp(-i k_r (dx cos psi_j + dy sin psi_j)), (dx, dy) in {-sqrt2, 0, +sqrt2}^2 px, px = 2/N,
  applied after the noise.
* Seeds: numpy SeedSequence([220207235, cfg]) spawned into six children (molecule, views,
  image->template choice, in-plane angles, noise, pair sample).  Bulk noise uses a
  counter-based splitmix64 hash evaluated with int64 torch ops, so CPU and CUDA generation
  draw the same uniforms for the same (seed, counter).

All evaluation is fp64 torch on the requested device; rings are returned as complex64
(the library's storage type) unless `complex128=True`.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import scipy.special
import torch

BASE_SEED = 220207235

# BASELINE.json "configs", in order (cfg index = position).
CONFIGS = {
    "tiny": dict(cfg=0, N=32, R=16, Q=64, T=8, M=8, atoms=20, snr=1.0, H=[4], views="random",
                 mol_cfg=0),
    "small": dict(cfg=1, N=64, R=32, Q=128, T=1024, M=1024, atoms=40, snr=0.5, H=[8],
                  views="fibonacci", mol_cfg=1),
    "medium": dict(cfg=2, N=128, R=64, Q=256, T=4096, M=4096, atoms=80, snr=0.1,
                   H=[64, 32, 16, 8], views="fibonacci", mol_cfg=2),
    "large": dict(cfg=3, N=256, R=128, Q=512, T=8192, M=16384, atoms=150, snr=0.05, H=[24],
                  views="fibonacci", mol_cfg=3),
    # G19: Translations reuses Medium's molecule (80 atoms), SNR 0.1 and Fibonacci views.
    "translations": dict(cfg=4, N=128, R=64, Q=256, T=2048, M=4096, atoms=80, snr=0.1, H=[16],
                         views="fibonacci", mol_cfg=2, shifts=9),
}

ATOM_SIGMA = 0.05
BALL_RADIUS = 0.3


def seed_children(cfg: int):
    """Six SeedSequence children: molecule, views, img->tmpl, angles, noise, pair sample."""
    return np.random.SeedSequence([BASE_SEED, cfg]).spawn(6)


def radial_grid(R: int):
    """Gauss-Jacobi(0,1) radial quadrature for k dk on [0, K], K = R-1 (G12).

    Returns (k, w) as float64 numpy arrays of length R.
    """
    if R < 1:
        raise ValueError("R must be >= 1")
    t, om = scipy.special.roots_jacobi(R, 0.0, 1.0)
    K = float(R - 1) if R > 1 else 1.0
    k = K * (t + 1.0) / 2.0
    w = (K * K / 4.0) * om
    return k.astype(np.float64), w.astype(np.float64)


def molecule_centres(cfg: int, n_atoms: int) -> np.ndarray:
    rng = np.random.default_rng(seed_children(cfg)[0])
    d = rng.standard_normal((n_atoms, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    rad = BALL_RADIUS * rng.random(n_atoms) ** (1.0 / 3.0)
    return d * rad[:, None]


def view_frames(cfg: int, T: int, scheme: str):
    """In-plane frames (e1, e2), each [T, 3] float64 (G14)."""
    if scheme == "fibonacci":
        i = np.arange(T, dtype=np.float64)
        z = 1.0 - (2.0 * i + 1.0) / T
        phi = i * math.pi * (3.0 - math.sqrt(5.0))
    elif scheme == "random":
        rng = np.random.default_rng(seed_children(cfg)[1])
        z = rng.uniform(-1.0, 1.0, T)
        phi = rng.uniform(0.0, 2.0 * math.pi, T)
    else:
        raise ValueError(scheme)
    th = np.arccos(np.clip(z, -1.0, 1.0))
    e1 = np.stack([np.cos(th) * np.cos(phi), np.cos(th) * np.sin(phi), -np.sin(th)], axis=1)
    e2 = np.stack([-np.sin(phi), np.cos(phi), np.zeros_like(phi)], axis=1)
    return e1, e2


# ---------------------------------------------------------------- counter-based normals
_M64 = (1 << 64) - 1


def _s64(x: int) -> int:
    x &= _M64
    return x - (1 << 64) if x >= (1 << 63) else x


def _srl(z: torch.Tensor, s: int) -> torch.Tensor:
    return (z >> s) & ((1 << (64 - s)) - 1)


def _mix64(z: torch.Tensor) -> torch.Tensor:
    z = z + _s64(0x9E3779B97F4A7C15)
    z = (z ^ _srl(z, 30)) * _s64(0xBF58476D1CE4E5B9)
    z = (z ^ _srl(z, 27)) * _s64(0x94D049BB133111EB)
    return z ^ _srl(z, 31)


def _mix64_py(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & _M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _M64
    return x ^ (x >> 31)


def counter_uniform(seed: int, counter: torch.Tensor) -> torch.Tensor:
    """Uniform(0,1) float64 from (seed, int64 counter) via splitmix64."""
    z = _mix64(counter + _s64(_mix64_py(seed)))
    return (_srl(z, 11).to(torch.float64) + 0.5) * (2.0 ** -53)


def counter_complex_normal(seed: int, start: int, n: int, device) -> torch.Tensor:
    """n standard complex normals (E|z|^2 = 1) for counters start..start+n-1 (Box-Muller)."""
    c = torch.arange(start, start + n, dtype=torch.int64, device=device)
    u1 = counter_uniform(seed, 2 * c)
    u2 = counter_uniform(seed, 2 * c + 1)
    rad = torch.sqrt(-2.0 * torch.log(u1))
    ang = 2.0 * math.pi * u2
    return torch.complex(rad * torch.cos(ang), rad * torch.sin(ang)) * (1.0 / math.sqrt(2.0))


# ---------------------------------------------------------------- analytic slices
def _slice_rows(p1: torch.Tensor, p2: torch.Tensor, gamma: torch.Tensor, k: torch.Tensor,
                Q: int) -> torch.Tensor:
    """B(k_r, psi_j - gamma_n) for rows n with projected atom coords p1, p2 [n, atoms].

    Returns complex128 [n, R, Q].
    """
    dev = p1.device
    psi = torch.arange(Q, dtype=torch.float64, device=dev) * (2.0 * math.pi / Q)
    ang = psi[None, :] - gamma[:, None]                      # [n, Q]
    c, s = torch.cos(ang), torch.sin(ang)
    g = torch.exp(-0.5 * (ATOM_SIGMA ** 2) * k * k)          # [R]
    n, R = p1.shape[0], k.shape[0]
    acc_re = torch.zeros((n, R, Q), dtype=torch.float64, device=dev)
    acc_im = torch.zeros((n, R, Q), dtype=torch.float64, device=dev)
    for a in range(p1.shape[1]):
        u = p1[:, a, None] * c + p2[:, a, None] * s           # [n, Q]
        ph = k[None, :, None] * u[:, None, :]                 # [n, R, Q]
        acc_re += torch.cos(ph)
        acc_im -= torch.sin(ph)
    out = torch.complex(acc_re, acc_im)
    return out * g[None, :, None]


def _rows_per_chunk(R: int, Q: int, device) -> int:
    budget = (1 << 25) if torch.device(device).type == "cuda" else (1 << 22)
    return max(1, budget // (R * Q))


@dataclass
class Dataset:
    name: str
    R: int
    Q: int
    N: int
    k: torch.Tensor                 # fp64 [R]
    w: torch.Tensor                 # fp64 [R]
    templates: torch.Tensor         # complex [T_local][R][Q]
    images: torch.Tensor            # complex [M_rows][R][Q]
    t_true: torch.Tensor            # int64 [M_rows], global template index of the source view
    gamma: torch.Tensor             # fp64 [M_rows], planted in-plane angle
    shift: torch.Tensor             # fp64 [M_rows, 2], translation (px units of box) or zeros
    sigma_hat2: float
    t_range: tuple = (0, 0)
    meta: dict = field(default_factory=dict)


def make_dataset(name: str, device="cpu", *, M: int | None = None, T: int | None = None,
                 t_range: tuple | None = None, complex128: bool = False,
                 snr: float | None = None, noise: bool = True) -> Dataset:
    """Build a config's inputs.  `M`/`T` override the counts (parity tests use reduced sizes);
    `t_range=(t0, t1)` returns only templates [t0, t1) (a rank's shard) while images still
    reference the full template set."""
    c = dict(CONFIGS[name])
    R, Q, N = c["R"], c["Q"], c["N"]
    T_all = T if T is not None else c["T"]
    M_base = M if M is not None else c["M"]
    snr = c["snr"] if snr is None else snr
    dev = torch.device(device)
    kk, ww = radial_grid(R)
    k = torch.tensor(kk, dtype=torch.float64, device=dev)
    w = torch.tensor(ww, dtype=torch.float64, device=dev)
    centres = torch.tensor(molecule_centres(c["mol_cfg"], c["atoms"]), device=dev)
    e1, e2 = view_frames(c["cfg"], T_all, c["views"])
    e1 = torch.tensor(e1, device=dev)
    e2 = torch.tensor(e2, device=dev)
    P1 = e1 @ centres.T                                       # [T, atoms]
    P2 = e2 @ centres.T
    ch = seed_children(c["cfg"])
    rng_t = np.random.default_rng(ch[2])
    rng_g = np.random.default_rng(ch[3])
    t_true = rng_t.integers(0, T_all, M_base)
    gam = rng_g.uniform(0.0, 2.0 * math.pi, M_base)
    noise_seed = int(ch[4].generate_state(1, dtype=np.uint64)[0])
    cdt = torch.complex128 if complex128 else torch.complex64
    step = _rows_per_chunk(R, Q, dev)

    t0, t1 = t_range if t_range is not None else (0, T_all)
    tmpl = torch.empty((t1 - t0, R, Q), dtype=cdt, device=dev)
    for s in range(t0, t1, step):
        e = min(t1, s + step)
        z = torch.zeros(e - s, dtype=torch.float64, device=dev)
        tmpl[s - t0:e - t0] = _slice_rows(P1[s:e], P2[s:e], z, k, Q).to(cdt)

    # images: signal, then noise calibrated on the mean signal power (G11)
    tt = torch.tensor(t_true, device=dev)
    gg = torch.tensor(gam, dtype=torch.float64, device=dev)
    imgs = torch.empty((M_base, R, Q), dtype=cdt, device=dev)
    dpsi = 2.0 * math.pi / Q
    power = torch.zeros((), dtype=torch.float64, device=dev)
    for s in range(0, M_base, step):
        e = min(M_base, s + step)
        sig = _slice_rows(P1[tt[s:e]], P2[tt[s:e]], gg[s:e], k, Q)
        power += ((sig.real ** 2 + sig.imag ** 2) * (w * dpsi)[None, :, None]).sum()
        imgs[s:e] = sig.to(cdt)
    pbar = float(power) / M_base
    sigma_hat2 = pbar / (snr * R * Q) if noise else 0.0
    node_sd = torch.sqrt(sigma_hat2 / (w * dpsi))              # [R]
    if noise and sigma_hat2 > 0:
        for s in range(0, M_base, step):
            e = min(M_base, s + step)
            nz = counter_complex_normal(noise_seed, s * R * Q, (e - s) * R * Q, dev)
            imgs[s:e] = (imgs[s:e].to(torch.complex128)
                         + nz.view(e - s, R, Q) * node_sd[None, :, None]).to(cdt)
    shift = torch.zeros((M_base, 2), dtype=torch.float64, device=dev)
    meta = dict(c, T=T_all, M=M_base, pbar=pbar, noise_seed=noise_seed)

    if c.get("shifts", 0) == 9:
        px = 2.0 / N
        d = [-math.sqrt(2.0) * px, 0.0, math.sqrt(2.0) * px]
        sh = torch.tensor([(dx, dy) for dx in d for dy in d], dtype=torch.float64, device=dev)
        psi = torch.arange(Q, dtype=torch.float64, device=dev) * dpsi
        rows = torch.empty((M_base * 9, R, Q), dtype=cdt, device=dev)
        for s in range(9):
            u = sh[s, 0] * torch.cos(psi) + sh[s, 1] * torch.sin(psi)        # [Q]
            ramp = torch.polar(torch.ones((R, Q), dtype=torch.float64, device=dev),
                               -(k[:, None] * u[None, :]))                   # [R, Q]
            for a in range(0, M_base, step):
                b = min(M_base, a + step)
                rows[a * 9 + s:b * 9 + s:9] = (imgs[a:b].to(torch.complex128) * ramp).to(cdt)
        imgs = rows
        tt = tt.repeat_interleave(9)
        gg = gg.repeat_interleave(9)
        shift = sh.repeat(M_base, 1)
        meta["M_rows"] = M_base * 9

    return Dataset(name=name, R=R, Q=Q, N=N, k=k, w=w, templates=tmpl, images=imgs,
                   t_true=tt, gamma=gg, shift=shift, sigma_hat2=sigma_hat2,
                   t_range=(t0, t1), meta=meta)


def toy_ctf(k, lam: float) -> np.ndarray:
    """Radial toy contrast-transfer function c(k) = -sin(pi lam k^2 / 2) (SPEC.md design decision:
    sign-oscillating contrast; real per-micrograph CTFs are out of scope).  Input model for row f3."""
    k = np.asarray(k.cpu() if torch.is_tensor(k) else k, dtype=np.float64)
    return -np.sin(np.pi * lam * k * k / 2.0)


def sample_pairs(name: str, M: int, T: int, n_random: int, n_true: int, t_true=None):
    """Seeded (m, t) pair sample: n_random uniform pairs plus n_true (m, t*(m)) pairs."""
    rng = np.random.default_rng(seed_children(CONFIGS[name]["cfg"])[5])
    m = rng.integers(0, M, n_random)
    t = rng.integers(0, T, n_random)
    if n_true and t_true is not None:
        mt = rng.integers(0, M, n_true)
        tt = np.asarray(t_true)[mt]
        m = np.concatenate([m, mt])
        t = np.concatenate([t, tt])
    return m.astype(np.int64), t.astype(np.int64)
