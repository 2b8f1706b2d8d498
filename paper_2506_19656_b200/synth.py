"""Seeded synthetic cubes with the shapes and value statistics of BASELINE.json's
five configurations (the real datasets are TB-scale and not available offline;
SURVEY.md §8d gives the generator recipes). Generated with torch on any device
(CPU for tests, the GPU for the benchmark); never timed.
"""

from __future__ import annotations

import math

import torch

CONFIGS = {
    1: dict(name="DeepExtremeCubes-shaped minicube", shape=(495, 128, 128, 7), dtype="f32",
            bit_depth=8, n_pcs=0, ssim=False, nan=True),
    2: dict(name="64 x DeepExtremeCubes minicube", shape=(495, 128, 128, 7), batch=64, dtype="f32",
            bit_depth=10, n_pcs=0, ssim=True, nan=True),
    3: dict(name="SimpleS2-shaped", shape=(64, 512, 512, 12), dtype="f32", bit_depth=12, n_pcs=9,
            ssim=True, nan=False),
    4: dict(name="DynamicEarthNet-shaped", shape=(730, 1024, 1024, 4), dtype="u16", bit_depth=8,
            n_pcs=0, ssim=False, nan=False),
    5: dict(name="ERA5-shaped", shape=(744, 721, 1440, 12), dtype="f32", bit_depth=16, n_pcs=6,
            ssim=True, nan=False, normalize=True),
}
SEEDS = {1: 19656, 2: 19656, 3: 29656, 4: 39656, 5: 49656}


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def smooth_field(h: int, w: int, sigma: float, gen, device, n: int = 1) -> torch.Tensor:
    """Gaussian-filtered N(0,1) noise (wrap boundaries), rescaled to unit std: [n,h,w]."""
    z = torch.randn((n, h, w), generator=gen, device=device, dtype=torch.float32)
    fy = torch.fft.fftfreq(h, device=device)
    fx = torch.fft.rfftfreq(w, device=device)
    k = torch.exp(-2 * (math.pi * sigma) ** 2 * (fy[:, None] ** 2 + fx[None, :] ** 2))
    f = torch.fft.irfft2(torch.fft.rfft2(z) * k, s=(h, w))
    f = f - f.mean(dim=(1, 2), keepdim=True)
    return f / f.std(dim=(1, 2), keepdim=True).clamp_min(1e-12)


def _ar1(T, shape, sigma, gen, device, rho=0.9):
    e = torch.randn(shape, generator=gen, device=device) * sigma
    yield e
    s = math.sqrt(1 - rho * rho) * sigma
    for _ in range(1, T):
        e = rho * e + s * torch.randn(shape, generator=gen, device=device)
        yield e


def minicube(seed: int, shape=(495, 128, 128, 7), device="cpu", nan: bool = True,
             period: float = 73.0, out: torch.Tensor | None = None) -> torch.Tensor:
    """Config 1/2: Sentinel-2-like reflectance in [0,1] with cloud NaNs."""
    T, H, W, C = shape
    g = _gen(seed, device)
    a = 0.05 + 0.30 * torch.rand(C, generator=g, device=device)
    A = 0.02 + 0.06 * torch.rand(C, generator=g, device=device)
    phi = 2 * math.pi * torch.rand(C, generator=g, device=device)
    S = smooth_field(H, W, 8.0, g, device, n=C).permute(1, 2, 0)  # [H,W,C]
    base = a + 0.05 * S
    cube = out if out is not None else torch.empty(shape, dtype=torch.float32, device=device)
    for t, e in enumerate(_ar1(T, (H, W, C), 0.02, g, device)):
        cube[t] = (base + A * torch.sin(2 * math.pi * t / period + phi) + e).clamp_(0.0, 1.0)
    if nan:
        n_nan_t = int(round(0.2 * T))
        tt = torch.randperm(T, generator=g, device=device)[:n_nan_t]
        cube[tt] = float("nan")
        keep = torch.ones(T, dtype=torch.bool, device=device)
        keep[tt] = False
        pix = torch.rand((T, H, W), generator=g, device=device) < 0.02
        pix &= keep[:, None, None]
        cube[pix] = float("nan")
    return cube


def minicube_batch(n: int, base_seed: int = 19656, shape=(495, 128, 128, 7), device="cpu",
                   nan: bool = True) -> torch.Tensor:
    out = torch.empty((n,) + tuple(shape), dtype=torch.float32, device=device)
    for b in range(n):
        minicube(base_seed + b, shape, device, nan, out=out[b])
    return out


def simple_s2(seed: int = 29656, shape=(64, 512, 512, 12), device="cpu", n_latent: int = 4):
    """Config 3: 4 latent minicube fields mixed into 12 correlated bands + 1% noise."""
    T, H, W, C = shape
    g = _gen(seed, device)
    lat = minicube(seed + 1, (T, H, W, n_latent), device, nan=False, period=12.0)
    M = torch.randn((n_latent, C), generator=g, device=device)
    out = torch.empty(shape, dtype=torch.float32, device=device)
    std = None
    for t in range(T):
        v = lat[t] @ M
        if std is None:
            std = v.reshape(-1, C).std(dim=0)
        out[t] = v + 0.01 * std * torch.randn((H, W, C), generator=g, device=device)
    return out


def dynamic_earthnet(seed: int = 39656, shape=(730, 1024, 1024, 4), device="cpu",
                     n_regions: int = 30, n_classes: int = 7) -> torch.Tensor:
    """Config 4: uint16 piecewise-constant land cover + daily AR(1) + 5% clouds at 10000."""
    T, H, W, C = shape
    g = _gen(seed, device)
    seeds = torch.rand((n_regions, 2), generator=g, device=device) * torch.tensor([H, W], device=device)
    yy, xx = torch.meshgrid(torch.arange(H, device=device), torch.arange(W, device=device), indexing="ij")
    pts = torch.stack([yy.reshape(-1), xx.reshape(-1)], dim=1).float()
    label = torch.cdist(pts, seeds).argmin(dim=1).reshape(H, W)
    cls = torch.randint(0, n_classes, (n_regions,), generator=g, device=device)[label]
    mu = 300 + 3700 * torch.rand((n_classes, C), generator=g, device=device)
    sd = 50 + 350 * torch.rand((n_classes, C), generator=g, device=device)
    static = mu[cls] + sd[cls] * torch.randn((H, W, C), generator=g, device=device)
    out = torch.empty(shape, dtype=torch.uint16, device=device)
    for t, e in enumerate(_ar1(T, (H, W, C), 100.0, g, device)):
        v = (static + e).clamp_(0, 10000).round_()
        cloud = torch.rand((H, W), generator=g, device=device) < 0.05
        v[cloud] = 10000
        out[t] = v.to(torch.int32).to(torch.uint16)
    return out


def era5(seed: int = 49656, shape=(744, 721, 1440, 12), device="cpu", t0: int = 0,
         out: torch.Tensor | None = None) -> torch.Tensor:
    """Config 5: lat-dependent mean + low-frequency field advected 1 px/hour,
    per-channel scale 10^(4c/11). ``t0`` selects a time slice of the cube."""
    T, H, W, C = shape
    g = _gen(seed, device)
    lat = torch.linspace(90.0, -90.0, H, device=device) * (math.pi / 180.0)
    F = smooth_field(H, W, min(40.0, W / 16.0), g, device, n=C).permute(1, 2, 0)  # [H,W,C]
    scale = torch.tensor([10 ** (4 * c / 11) for c in range(C)], device=device, dtype=torch.float32)
    base = 1.5 + 0.5 * torch.cos(lat)[:, None, None]
    res = out if out is not None else torch.empty(shape, dtype=torch.float32, device=device)
    for t in range(T):
        Ft = torch.roll(F, shifts=t0 + t, dims=1)
        res[t] = scale * (base + 0.3 * Ft)
    return res


def make(config: int, device="cpu", batch: int | None = None, T: int | None = None,
         spatial: tuple | None = None) -> torch.Tensor:
    """Generate a configuration's cube(s), optionally truncated in T / space (tests)."""
    cfg = CONFIGS[config]
    shape = list(cfg["shape"])
    if T is not None:
        shape[0] = T
    if spatial is not None:
        shape[1], shape[2] = spatial
    shape = tuple(shape)
    if config == 1:
        return minicube(SEEDS[1], shape, device)
    if config == 2:
        return minicube_batch(batch or cfg["batch"], SEEDS[2], shape, device)
    if config == 3:
        return simple_s2(SEEDS[3], shape, device)
    if config == 4:
        return dynamic_earthnet(SEEDS[4], shape, device)
    return era5(SEEDS[5], shape, device)
