"""Seeded synthetic volumes (spherical-harmonic shells) for row f4 (volume alignment).

HARNESS, not method: produces the inputs both the CUDA path and the oracle consume.  It holds none
of the alignment arithmetic (no kernels, bases, Wigner-d, inner products).

Recipe (the paper's volumes -- de-novo TRPV1 reconstructions and
emd-5778, PAPER.md:1051-1060 -- are not available, so phantoms stand in for them):

* Radial grid: R Gauss-Jacobi(alpha=0, beta=2) nodes t_r on [-1, 1] mapped by
  k = K (t + 1) / 2, weights w_r = (K/2)^3 omega_r, so sum_r g(k_r) w_r ~ int_0^K g(k) k^2 dk.
* Phantom: n_atoms isotropic Gaussian atoms (sigma = 0.05), centres uniform in the ball of radius
  rho = 0.3, amplitude 1.  Its Fourier transform sum_a exp(-sigma^2 k^2 / 2) exp(-i k . c_a) has the
  spherical-harmonic coefficients (plane-wave expansion)
      A_l^m(k) = sum_a exp(-sigma^2 k^2 / 2) 4 pi (-i)^l j_l(k |c_a|) conj(Y_l^m(c_a / |c_a|)),
  Y_l^m orthonormal with the Condon-Shortley phase (scipy.special.sph_harm_y), truncated at l <= L
  (packed lm = l^2 + l + m).  K defaults to L / (4 rho) so the truncation error is ~(e/8)^L.
* Volumes to align (many volumes, one target): volume n is the target's atoms
  jittered by N(0, jitter^2) per coordinate and rotated by tau_n = (gamma, beta, alpha) on the
  alignment grid, centres c -> R_z(alpha) R_y(beta) R_z(gamma) c, i.e. the
  volume R_tau B.
* Grids: alpha_a = 2 pi a / P, gamma_g = 2 pi g / P (PAPER.md:890 with P points, DESIGN.md reading
  V1), beta_b = -pi + 2 pi b / nb on [-pi, pi) ("a grid of M different beta-values").
* Seeds: numpy SeedSequence([220207235, 4, seed]) -> (target atoms, jitter, rotations).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.special

BASE_SEED = 220207235


def radial_grid_k2(R: int, K: float):
    t, om = scipy.special.roots_jacobi(R, 0.0, 2.0)
    return K * (t + 1.0) / 2.0, (K / 2.0) ** 3 * om


def rotation(alpha: float, beta: float, gamma: float) -> np.ndarray:
    """R_tau = R^z_alpha R^y_beta R^z_gamma."""
    def rz(a):
        return np.array([[np.cos(a), -np.sin(a), 0.0], [np.sin(a), np.cos(a), 0.0], [0.0, 0.0, 1.0]])
    ry = np.array([[np.cos(beta), 0.0, np.sin(beta)], [0.0, 1.0, 0.0], [-np.sin(beta), 0.0, np.cos(beta)]])
    return rz(alpha) @ ry @ rz(gamma)


def sh_coefficients(centres: np.ndarray, k: np.ndarray, L: int, sigma: float = 0.05,
                    amps: np.ndarray | None = None) -> np.ndarray:
    """[R, (L+1)^2] complex128 coefficients of sum_a amp_a exp(-sigma^2 k^2/2) exp(-i k . c_a)."""
    c = np.asarray(centres, np.float64)
    amps = np.ones(len(c)) if amps is None else np.asarray(amps, np.float64)
    rad = np.linalg.norm(c, axis=1)
    theta = np.arccos(np.clip(c[:, 2] / np.maximum(rad, 1e-300), -1.0, 1.0))
    phi = np.arctan2(c[:, 1], c[:, 0])
    out = np.zeros((len(k), (L + 1) ** 2), np.complex128)
    damp = np.exp(-0.5 * sigma ** 2 * k ** 2)
    for l in range(L + 1):
        jl = scipy.special.spherical_jn(l, np.outer(k, rad))               # [R, atoms]
        for m in range(-l, l + 1):
            y = np.conj(scipy.special.sph_harm_y(l, m, theta, phi))       # [atoms]
            out[:, l * l + l + m] = 4.0 * np.pi * (-1j) ** l * damp * (jl @ (amps * y))
    return out


def gaussian_overlap(centres_a, centres_b, k, w, sigma: float = 0.05) -> float:
    """sum_r w_r int_{S^2} conj(A(k_r, khat)) B(k_r, khat) dkhat for two Gaussian-atom phantoms in closed
    form, 4 pi sum_{a,b} exp(-sigma^2 k^2) j_0(k |c_a - c_b|) (a test pin, not the method)."""
    d = np.linalg.norm(np.asarray(centres_a)[:, None, :] - np.asarray(centres_b)[None, :, :], axis=-1)
    kr = np.asarray(k)[:, None, None] * d[None]
    return float(np.sum(np.asarray(w) * np.exp(-sigma ** 2 * np.asarray(k) ** 2)
                        * 4.0 * np.pi * np.sum(np.sinc(kr / np.pi), axis=(1, 2))))


def beta_grid(nb: int) -> np.ndarray:
    return -np.pi + 2.0 * np.pi * np.arange(nb) / nb


def ball_points(rng, n: int, rho: float) -> np.ndarray:
    v = rng.standard_normal((n, 3))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    return v * rho * rng.random(n)[:, None] ** (1.0 / 3.0)


@dataclass
class VolumeSet:
    L: int
    R: int
    K: float
    k: np.ndarray
    w: np.ndarray
    P: int
    betas: np.ndarray
    target: np.ndarray          # [R, (L+1)^2] complex64
    volumes: np.ndarray         # [n, R, (L+1)^2] complex64
    target_centres: np.ndarray
    tau_index: np.ndarray       # [n, 3] (b, a, g) of the rotation applied to volume n


def grid_size(L: int) -> int:
    """P = smallest power of two >= max(32, 2L + 1) (reading V1)."""
    P = 32
    while P < 2 * L + 1:
        P *= 2
    return P


def make_volumes(L: int, R: int, n: int, nb: int | None = None, atoms: int = 40, rho: float = 0.3,
                 sigma: float = 0.05, jitter: float = 0.0, K: float | None = None, seed: int = 0,
                 P: int | None = None) -> VolumeSet:
    P = P or grid_size(L)
    nb = nb or (2 * L + 1)
    K = K if K is not None else L / (4.0 * rho)
    k, w = radial_grid_k2(R, K)
    ss = np.random.SeedSequence([BASE_SEED, 4, seed]).spawn(3)
    r_atoms, r_jit, r_rot = (np.random.default_rng(s) for s in ss)
    centres = ball_points(r_atoms, atoms, rho)
    target = sh_coefficients(centres, k, L, sigma)
    betas = beta_grid(nb)
    tau = np.stack([r_rot.integers(0, nb, n), r_rot.integers(0, P, n), r_rot.integers(0, P, n)], axis=1)
    vols = np.empty((n, R, (L + 1) ** 2), np.complex128)
    for i in range(n):
        b, a, g = tau[i]
        c = centres + jitter * r_jit.standard_normal(centres.shape)
        Rm = rotation(2 * np.pi * a / P, betas[b], 2 * np.pi * g / P)
        vols[i] = sh_coefficients(c @ Rm.T, k, L, sigma)
    return VolumeSet(L, R, K, k, w, P, betas, target.astype(np.complex64), vols.astype(np.complex64),
                     centres, tau)
