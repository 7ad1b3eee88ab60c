"""Synthetic smooth fields for tests and the benchmark (SURVEY §8d inputs).

Not part of the compress/decompress path.  Kinds:
  grf    Gaussian random field, isotropic Fourier amplitude k^(-11/6) *
         exp(-(k/0.08)^2) (Kolmogorov-like inertial range with a resolved
         dissipation cutoff), normalised to [0, 1] -- the headline input.
  rough  white noise filtered by 1/(1 + k^2/0.005), normalised to [0, 1]
         (rough, outlier-producing stress case).
  gauss  sum of six random anisotropic Gaussians (very smooth).
  modes  random-phase spectral synthesis (turbulence-like): a sum
         of separable Fourier modes with a k^(-11/6) exp(-(k/0.08)^2) amplitude,
         defined per GLOBAL coordinate, so any axis-0 slab of a huge volume
         (config 5: 2048^3) is generated on its own GPU without the rest.
`make` builds host numpy arrays, `make_device` builds torch CUDA tensors with
the same recipe (values differ between the two; each is deterministic).
"""

from __future__ import annotations

import numpy as np


def _dims3(dims):
    d = tuple(int(x) for x in dims)
    return d + (1,) if len(d) == 2 else d


def _k2(xp, d, rfft_last=True):
    ks = []
    for a, n in enumerate(d):
        if a == 2 and rfft_last:
            k = xp.fft.rfftfreq(n)
        else:
            k = xp.fft.fftfreq(n)
        shape = [1, 1, 1]
        shape[a] = k.shape[0]
        ks.append(k.reshape(shape))
    return ks[0] ** 2 + ks[1] ** 2 + ks[2] ** 2


def _normalise(v):
    lo, hi = v.min(), v.max()
    return (v - lo) / (hi - lo) if hi > lo else v * 0


def make(kind: str, dims, seed: int = 0, dtype="f32") -> np.ndarray:
    d = _dims3(dims)
    rng = np.random.default_rng(seed)
    if kind in ("grf", "rough"):
        noise = rng.standard_normal(d)
        spec = np.fft.rfftn(noise)
        k2 = _k2(np, d)
        if kind == "grf":
            k = np.sqrt(k2)
            with np.errstate(divide="ignore"):
                amp = np.where(k > 0, k ** (-11.0 / 6.0), 0.0) * np.exp(-(k / 0.08) ** 2)
        else:
            amp = 1.0 / (1.0 + k2 / 0.005)
        v = np.fft.irfftn(spec * amp, s=d, axes=(0, 1, 2))
        v = _normalise(v)
    elif kind == "gauss":
        x = [np.arange(n, dtype=np.float64).reshape([-1 if a == i else 1 for i in range(3)]) for a, n in enumerate(d)]
        c = rng.uniform(0, 1, (6, 3)) * np.array(d)
        s = rng.uniform(0.08, 0.35, (6, 3)) * np.maximum(np.array(d, np.float64), 2.0)
        amp = rng.uniform(0.2, 1.0, 6)
        v = np.zeros(d)
        for i in range(6):
            v += amp[i] * np.exp(-0.5 * sum(((x[a] - c[i, a]) / s[i, a]) ** 2 for a in range(3)))
    else:
        raise ValueError(kind)
    return np.ascontiguousarray(v.astype(np.float32 if dtype in ("f32", np.float32) else np.float64))


def make_device(kind: str, dims, seed: int = 0, dtype="f32", device="cuda"):
    """Same recipes on the GPU with torch (fast at 512^3 and for slabs)."""
    import torch
    d = _dims3(dims)
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    if kind in ("grf", "rough"):
        noise = torch.randn(d, generator=g, device=device, dtype=torch.float64)
        spec = torch.fft.rfftn(noise)
        del noise
        k2 = _k2(torch, d).to(device)
        if kind == "grf":
            k = torch.sqrt(k2)
            amp = torch.where(k > 0, k.clamp_min(1e-30) ** (-11.0 / 6.0), torch.zeros_like(k)) * torch.exp(-(k / 0.08) ** 2)
        else:
            amp = 1.0 / (1.0 + k2 / 0.005)
        spec *= amp
        v = torch.fft.irfftn(spec, s=d, dim=(0, 1, 2))
        del spec
        lo, hi = v.min(), v.max()
        v = (v - lo) / (hi - lo)
    elif kind == "gauss":
        dd = torch.tensor(d, dtype=torch.float64)
        c = torch.rand((6, 3), generator=torch.Generator().manual_seed(seed), dtype=torch.float64) * dd
        s = (0.08 + 0.27 * torch.rand((6, 3), generator=torch.Generator().manual_seed(seed + 1),
                                      dtype=torch.float64)) * dd.clamp_min(2.0)
        amp = 0.2 + 0.8 * torch.rand(6, generator=torch.Generator().manual_seed(seed + 2), dtype=torch.float64)
        x = [torch.arange(n, dtype=torch.float64, device=device).reshape([-1 if a == i else 1 for i in range(3)])
             for a, n in enumerate(d)]
        v = torch.zeros(d, dtype=torch.float64, device=device)
        for i in range(6):
            v += amp[i].item() * torch.exp(-0.5 * sum(((x[a] - c[i, a].item()) / s[i, a].item()) ** 2
                                                      for a in range(3)))
    else:
        raise ValueError(kind)
    return v.to(torch.float32 if dtype in ("f32", np.float32) else torch.float64).contiguous()


def _mode_tables(global_dims, seed: int, n_modes: int):
    """Per-mode wave numbers, phases and amplitudes (host, tiny; numpy RNG)."""
    d = np.array(_dims3(global_dims), np.float64)
    rng = np.random.default_rng(seed)
    # integer wave numbers (periodic over the global box), |k| log-uniform
    # between the box scale and the 0.08 cycles/point cutoff
    kmag = np.exp(rng.uniform(np.log(1.0 / d.max()), np.log(0.12), n_modes))
    u = rng.standard_normal((n_modes, 3))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    k = np.round(np.abs(u) * kmag[:, None] * d) / d  # cycles per point along each axis
    k = np.where(d[None, :] > 1, k, 0.0)
    kk = np.sqrt((k * k).sum(1))
    amp = np.where(kk > 0, np.maximum(kk, 1e-12) ** (-11.0 / 6.0), 0.0) * np.exp(-(kk / 0.08) ** 2)
    # density of the log-uniform |k| draw is 1/k: weight by k^(3/2) so the
    # sum approximates an isotropic k^-11/6 spectrum in 3D
    amp *= kk ** 1.5
    amp /= np.sqrt((amp * amp).sum()) + 1e-300
    phase = rng.uniform(0, 2 * np.pi, (n_modes, 3))
    return k, phase, amp


def make_modes(dims, seed: int = 0, dtype="f32", x0: int = 0, global_dims=None, n_modes: int = 96,
               device="cuda"):
    """Rows [x0, x0 + dims[0]) of the global `modes` field, on the GPU.

    v(x, y, z) = sum_m a_m cos(2 pi kx_m x + px_m) cos(2 pi ky_m y + py_m) cos(2 pi kz_m z + pz_m)
    evaluated as one (ny, M) x (M, nz) GEMM per x-plane (fp32 or fp64 cuBLAS,
    TF32 off), so the value at a global coordinate never depends on the slab
    that contains it."""
    import torch
    d = _dims3(dims)
    gd = _dims3(global_dims) if global_dims is not None else d
    k, ph, amp = _mode_tables(gd, seed, n_modes)
    tdt = torch.float32 if dtype in ("f32", np.float32) else torch.float64

    def axis(a, lo, n):
        c = torch.arange(lo, lo + n, dtype=torch.float64, device=device)
        kt = torch.tensor(k[:, a], dtype=torch.float64, device=device)
        pt = torch.tensor(ph[:, a], dtype=torch.float64, device=device)
        return torch.cos(2 * np.pi * kt[:, None] * c[None, :] + pt[:, None])  # (M, n)

    A = axis(0, x0, d[0]) * torch.tensor(amp, dtype=torch.float64, device=device)[:, None]
    B = axis(1, 0, d[1]).to(tdt)
    C = axis(2, 0, d[2]).to(tdt)
    A = A.to(tdt)
    out = torch.empty(d, dtype=tdt, device=device)
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        Bt = B.t().contiguous()
        for i in range(d[0]):  # one GEMM shape for every plane of every slab
            torch.mm(Bt * A[:, i][None, :], C, out=out[i])
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    return out
