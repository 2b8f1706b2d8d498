"""The fused array path: encode-prep (frames for the codec) and decode + score.

Follows the composition order of the reference's (absent) container,
SPEC.md:351 (compress) and SPEC.md:360 (decompress):

  encode_prep : select -> forward fill (+mask) -> [pca_fit -> pca_forward]
                -> fit_quant -> quantize -> pack_groups -> planar frames
  decode_eval : frames -> drop padded planes -> dequantize -> [pca_inverse]
                -> recon, scored against the (filled) original

Non-PCA streams run as three kernels with no host synchronisation
(K1 stats+carries, K4 fill+quantise+pack, K5/K6 decode+PSNR+SSIM); PCA streams
add the float64 Gram pass, one host ``eigh`` (C x C) and the projection pass.
Cubes are ``[T,H,W,C]`` or batches ``[B,T,H,W,C]`` (independent cubes, one
QuantParams each), numpy or CUDA tensors.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device as dev
from . import _lib
from .bridge import check_stream_bytes
from .errors import ConfigurationError, CorruptStreamError
from .metrics import SSIM_WINDOW, psnr_from_sse
from .plan import pack_groups
from .transform import (SUPPORTED_BIT_DEPTHS, PcaModel, QuantParams, band_stats,
                        covariance_from_gram, eig_model, gram)

_PAD = {"repeat": _lib.CV_PAD_REPEAT, "zero": _lib.CV_PAD_ZERO}


@dataclass(frozen=True)
class StreamSpec:
    """The MappingRule fields that matter to the array path (plan.py:26-44)."""

    bit_depth: int
    n_pcs: int = 0
    fill_value: float = 0.0          # MappingRule.fill_value_for_leading
    normalize: bool = False          # per-band min/max normalisation before PCA
    clamp: bool = False
    pad_mode: str = "repeat"         # plan.py:126 ("zero" is BASELINE's wording)
    seg_len: int = 16                # time steps per CTA (forward-fill carry granularity)

    def __post_init__(self):
        if self.bit_depth not in SUPPORTED_BIT_DEPTHS:
            raise ConfigurationError(f"bit depth {self.bit_depth} not in {SUPPORTED_BIT_DEPTHS}")
        if self.pad_mode not in _PAD:
            raise ConfigurationError(f"pad_mode must be one of {sorted(_PAD)}")
        if self.n_pcs < 0:
            raise ConfigurationError("n_pcs must be >= 0")


@dataclass
class PcaFold:
    """A PcaModel (possibly in normalised space) folded into kernel constants."""

    model: PcaModel
    fwd_mean: np.ndarray
    fwd_comps: np.ndarray
    inv_mean: np.ndarray
    inv_comps: np.ndarray
    norm_offset: np.ndarray | None = None
    norm_scale: np.ndarray | None = None


@dataclass
class Encoded:
    """Frames plus everything decode needs (the manifest's array part)."""

    frames: torch.Tensor                 # [B][G][T][3][H*W] u8 / u16
    qmins: torch.Tensor                  # [B][E] float64 (device)
    qmaxs: torch.Tensor
    spec: StreamSpec
    shape: tuple                         # (B, T, H, W, C)
    groups: list
    peaks: torch.Tensor                  # [B][C] max of the (filled) original
    nan_counts: torch.Tensor | None      # [B][C] synthesised cells
    seg_last: torch.Tensor | None        # forward-fill carry map (scoring the filled cube)
    pca: list = field(default_factory=list)   # one PcaFold per cube
    err: dev.ErrWord | None = None
    filled: torch.Tensor | None = None   # forward-filled cube (float32 sources)
    t_total: int | None = None           # frames over all time shards (multi-GPU)
    shard: object | None = None          # dist.TimeShard of a time-sharded stream

    @property
    def n_encoded(self) -> int:
        return self.qmins.shape[1]

    @property
    def frame_bytes(self) -> int:
        return self.frames.numel() * self.frames.element_size()

    def quant_params(self, cube: int = 0) -> QuantParams:
        return QuantParams(self.spec.bit_depth, tuple(self.qmins[cube].tolist()),
                           tuple(self.qmaxs[cube].tolist()))

    def check(self) -> None:
        """Read the error word once and raise like the reference would."""
        if self.err is None:
            return
        f = self.err.flags()
        if f & _lib.CV_FLAG_NONFINITE:
            raise ConfigurationError("array contains +/-inf; only NaN marks missing data")
        if f & _lib.CV_FLAG_NAN:
            raise ConfigurationError("cannot fit quantization on non-finite values")
        if f & _lib.CV_FLAG_RANGE:
            raise ConfigurationError("values outside the quantization range (pass clamp=True to clip)")
        if f & _lib.CV_FLAG_INT_RANGE:
            raise ConfigurationError("integer values outside the bit-depth range")


class Workspace:
    """Reusable device buffers for repeated calls on same-shaped cubes (frames,
    filled cube, carry map, recon). Large allocations inside a hot loop make
    the caching allocator fall back to cudaMalloc/cudaFree (which synchronise
    the device) whenever fragmentation forbids a cached fit; a Workspace pins
    them once. Buffers handed out for one call are overwritten by the next."""

    def __init__(self):
        self._bufs = {}

    def get(self, name: str, shape, dtype, device) -> torch.Tensor:
        key = (name, tuple(shape), dtype, str(device))
        t = self._bufs.get(key)
        if t is None:
            t = torch.empty(tuple(shape), dtype=dtype, device=device)
            self._bufs[key] = t
        return t


def _alloc(ws: Workspace | None, name, shape, dtype, device) -> torch.Tensor:
    if ws is None:
        return torch.empty(tuple(shape), dtype=dtype, device=device)
    return ws.get(name, shape, dtype, device)


def _as_batch(cube) -> tuple[dev.Arr, tuple]:
    x = dev.to_device(cube)
    if len(x.shape) == 4:
        B, (T, H, W, C) = 1, x.shape
    elif len(x.shape) == 5:
        B, T, H, W, C = x.shape
    else:
        raise ConfigurationError(f"expected a [t,y,x,c] cube or a [b,t,y,x,c] batch, got {len(x.shape)}-D")
    if x.code is None:
        raise ConfigurationError(f"unsupported dtype {x.np_dtype} for the B200 path")
    return x, (B, T, H, W, C)


def _fold(model: PcaModel, offset=None, scale=None) -> PcaFold:
    W = np.ascontiguousarray(model.components, dtype=np.float64)
    mu = np.ascontiguousarray(model.mean, dtype=np.float64)
    if offset is None:
        return PcaFold(model, mu, W, mu, W)
    # z = (v - offset) / scale ; pc = (z - mu) W^T  ==  (v - (offset + scale*mu)) (W / scale)^T
    fwd_mean = offset + scale * mu
    fwd = W / scale[None, :]
    inv = W * scale[None, :]
    return PcaFold(model, np.ascontiguousarray(fwd_mean), np.ascontiguousarray(fwd),
                   np.ascontiguousarray(fwd_mean), np.ascontiguousarray(inv), offset, scale)


def _cube_view(x: dev.Arr, b: int, T: int, HW: int, C: int) -> dev.Arr:
    return dev.Arr(x.t[b] if x.t.dim() == 5 else x.t, x.code, x.host, x.np_dtype, (T, HW, C))


def _launch_grams(x: dev.Arr, B: int, T: int, HW: int, C: int, err: dev.ErrWord) -> list:
    """K2 (float64 shifted Gram + band min/max) of every cube; device-side only."""
    return [gram(_cube_view(x, b, T, HW, C), T * HW, C, stats=True, err=err) for b in range(B)]


def _fit_models(grams: list, n: int, C: int, n_pcs: int, normalize: bool, shard=None):
    """Gram partials -> host eigh -> folded models; one device->host copy for all cubes.

    With a multi-rank ``shard`` every rank re-centres the gathered partials on
    rank 0's shift, so all ranks fit the identical model.
    """
    sharded = shard is not None and shard.world > 1
    folds, peaks = [], []
    if not sharded:
        pack = torch.stack([torch.cat([g["shift"].double(), g["out"], g["mins"], g["maxs"]])
                            for g in grams]).cpu().numpy()
    for b, g in enumerate(grams):
        if sharded:
            shift, out, nn = shard.combine_gram(g["shift"], g["out"], n, C)
            gmins, gmaxs = shard.combine_minmax(g["mins"], g["maxs"])
            mins, maxs = gmins.cpu().numpy(), gmaxs.cpu().numpy()
            peaks.append(gmaxs)
        else:
            row = pack[b]
            shift, out = row[:C], row[C:2 * C + C * C]
            mins, maxs = row[2 * C + C * C:3 * C + C * C], row[3 * C + C * C:]
            nn = n
            peaks.append(g["maxs"])
        mean, cov = covariance_from_gram(shift, out, nn, C)
        if normalize:
            scale = maxs - mins
            scale = np.where(scale == 0, 1.0, scale)
            zmean = (mean - mins) / scale
            zcov = cov / np.outer(scale, scale)
            folds.append(_fold(eig_model(zmean, zcov, n_pcs, C), mins, scale))
        else:
            folds.append(_fold(eig_model(mean, cov, n_pcs, C)))
    return folds, torch.stack(peaks)


def _fill_stats(x: dev.Arr, spec: StreamSpec, B: int, T: int, HW: int, C: int, err: dev.ErrWord,
                workspace, shard):
    """K1 in fill mode (forward-fill carries + per-band ranges of the filled cube).

    Returns (qmins, qmaxs, nan_counts, seg_last, carry_in); in a time-sharded
    stream the ranges are global and ``carry_in`` holds the last observation
    of the earlier shards.
    """
    lib = _lib.load()
    d = x.device
    nseg = lib.cv_num_segments(T, spec.seg_len)
    seg_last = _alloc(workspace, "seg_last", (B, nseg, HW * C), torch.float32, d)
    if shard is None or shard.world == 1:
        qmins, qmaxs, nans = band_stats(x, B, T, HW * C, C, fill_mode=1, seg_len=spec.seg_len,
                                        fill_value=spec.fill_value, err=err, seg_last=seg_last)
        return qmins, qmaxs, nans, seg_last, None
    from .dist import last_observed, raw_band_stats

    mins, maxs, lead, nans = raw_band_stats(x, B, T, HW * C, C, 1, spec.seg_len, err, seg_last)
    qmins, qmaxs, nans = shard.combine_band_stats(mins, maxs, lead, nans, spec.fill_value)
    return qmins, qmaxs, nans, seg_last, shard.carry_in(last_observed(seg_last))


def encode_prep(cube, spec: StreamSpec, marks=None, filled_out: torch.Tensor | None = None,
                shard=None, workspace: Workspace | None = None) -> Encoded:
    """Cube(s) -> planar integer frames + QuantParams (+ PCA models).

    Float32 cubes are forward-filled (cube.py:213-246) before anything else
    sees them. Without PCA the fill is fused into the quantiser, which also
    writes the filled cube (``Encoded.filled``, forward_fill_time's output) so
    decode scores against what the codec saw. With PCA the Gram pass runs on
    the raw cube first; if it met NaN (every rank agrees through one
    all-reduce of the error flags) the cube is forward-filled into the
    workspace and the Gram, projection and quantiser read the filled copy,
    as the reference's pca_fit is fed the filled array (transform.py:160-188).
    ``marks`` (optional callable) is invoked with a phase label after the
    statistics phase (benchmark CUDA events).
    """
    x, (B, T, H, W, C) = _as_batch(cube)
    d = x.device
    HW = H * W
    s = dev.stream_ptr(d)
    err = dev.ErrWord(d)
    if x.t.numel() == 0:
        raise ConfigurationError("empty cube")
    fill = x.code == _lib.CV_F32
    seg = spec.seg_len
    lib = _lib.load()
    sharded = shard is not None and shard.world > 1
    carry_in = None
    filled = None
    if spec.n_pcs == 0:
        E = C
        seg_last = None
        if fill:
            qmins, qmaxs, nans, seg_last, carry_in = _fill_stats(x, spec, B, T, HW, C, err, workspace,
                                                                 shard)
        elif not sharded:
            qmins, qmaxs, nans = band_stats(x, B, T, HW * C, C, fill_mode=0, seg_len=seg, err=err)
        else:
            from .dist import raw_band_stats

            mins, maxs, lead, nans = raw_band_stats(x, B, T, HW * C, C, 0, seg, err, None)
            qmins, qmaxs, nans = shard.combine_band_stats(mins, maxs, lead, nans, spec.fill_value)
        peaks = qmaxs
        folds = []
        src = x
    else:
        if spec.n_pcs > C:
            raise ConfigurationError(f"n_keep={spec.n_pcs} outside [1, {C}]")
        E = spec.n_pcs
        seg_last, nans = None, None
        src = x
        gerr = dev.ErrWord(d)
        grams = _launch_grams(src, B, T, HW, C, gerr)
        flags = gerr.flags()
        if sharded:
            flags = shard.combine_flags(flags)
        if flags & _lib.CV_FLAG_NONFINITE:
            raise ConfigurationError("array contains +/-inf; only NaN marks missing data")
        if flags & _lib.CV_FLAG_NAN:
            if not fill:
                raise ConfigurationError("cannot fit a PCA on non-finite values")
            # fill (+mask) before pca_fit / pca_forward
            _, _, nans, seg_last, carry_in = _fill_stats(x, spec, B, T, HW, C, err, workspace, shard)
            filled = filled_out if filled_out is not None else _alloc(workspace, "filled", x.t.shape,
                                                                      x.t.dtype, d)
            _lib.call("cv_forward_fill", x.ptr, B, T, HW * C, float(spec.fill_value), seg,
                      seg_last.data_ptr(), carry_in.data_ptr() if carry_in is not None else None,
                      filled.data_ptr(), None, err.ptr, s)
            src = dev.Arr(filled, x.code, x.host, x.np_dtype, x.shape)
            gerr.reset()
            grams = _launch_grams(src, B, T, HW, C, gerr)
        folds, peaks = _fit_models(grams, T * HW, C, E, spec.normalize, shard)
        qmins = torch.empty((B, E), dtype=torch.float64, device=d)
        qmaxs = torch.empty_like(qmins)
        sws = dev.workspace(lib.cv_stats_ws_bytes(B, E), d)
        _lib.call("cv_stats_reset", sws.data_ptr(), B, E, s)
        esz = lib.cv_stats_ws_bytes(1, E)
        for b in range(B):
            fold = folds[b]
            _lib.call("cv_pca_project", _cube_view(src, b, T, HW, C).ptr, src.code, 1, T * HW, C,
                      fold.fwd_mean.ctypes.data, fold.fwd_comps.ctypes.data, E, None, _lib.CV_F64,
                      sws.data_ptr() + b * esz, err.ptr, s)
        _lib.call("cv_stats_finalize", sws.data_ptr(), B, E, 0, 0.0, qmins.data_ptr(),
                  qmaxs.data_ptr(), None, s)
        if sharded:
            qmins, qmaxs = shard.combine_minmax(qmins, qmaxs)
    if marks is not None:
        marks("stats")
    groups = pack_groups(E)
    G = len(groups)
    tdt, _ = dev.out_dtype_for_depth(spec.bit_depth)
    frames = _alloc(workspace, "frames", (B, G, T, 3, HW), tdt, d)
    if spec.n_pcs == 0:
        if fill:
            filled = filled_out if filled_out is not None else _alloc(workspace, "filled", x.t.shape,
                                                                      x.t.dtype, d)
        _lib.call("cv_quantize", x.ptr, x.code, B, T, HW, C, qmins.data_ptr(), qmaxs.data_ptr(),
                  spec.bit_depth, int(spec.clamp), int(fill), float(spec.fill_value), seg,
                  seg_last.data_ptr() if seg_last is not None else None,
                  carry_in.data_ptr() if carry_in is not None else None, None, None, 0,
                  _lib.CV_LAYOUT_PLANAR, _PAD[spec.pad_mode], frames.data_ptr(),
                  filled.data_ptr() if filled is not None else None, err.ptr, s)
    else:
        for b in range(B):
            fold = folds[b]
            _lib.call("cv_quantize", _cube_view(src, b, T, HW, C).ptr, src.code, 1, T, HW, C,
                      qmins[b:].data_ptr(), qmaxs[b:].data_ptr(), spec.bit_depth, int(spec.clamp), 0,
                      0.0, seg, None, None, fold.fwd_mean.ctypes.data, fold.fwd_comps.ctypes.data, E,
                      _lib.CV_LAYOUT_PLANAR, _PAD[spec.pad_mode], frames[b].data_ptr(), None,
                      err.ptr, s)
    enc = Encoded(frames, qmins, qmaxs, spec, (B, T, H, W, C), groups, peaks, nans, seg_last,
                  folds, err, filled)
    if sharded:
        tt = torch.tensor([T], dtype=torch.int64, device=d)
        shard.all_reduce(tt)
        enc.t_total = int(tt.item())
        enc.shard = shard
    return enc


@dataclass
class Scores:
    """Per-cube, per-band metric sums on the device; ``report()`` syncs once."""

    sse: torch.Tensor       # [B][C]
    ssim_sum: torch.Tensor  # [B][C] (zeros when SSIM was not requested)
    peaks: torch.Tensor     # [B][C]
    n_per_band: int
    n_ssim_per_band: int
    want_ssim: bool
    frame_bytes_per_cube: int
    shape: tuple

    def report(self) -> list:
        sse = self.sse.cpu().numpy()
        ssum = self.ssim_sum.cpu().numpy()
        peaks = self.peaks.cpu().numpy()
        B, T, H, W, C = self.shape
        out = []
        for b in range(sse.shape[0]):
            db, agg = psnr_from_sse(sse[b], peaks[b], self.n_per_band)
            rep = {"psnr_per_band": db, "psnr": agg,
                   "bpppb": 8.0 * self.frame_bytes_per_cube / (T * H * W * C)}
            if self.want_ssim:
                per = ssum[b] / self.n_ssim_per_band
                rep["ssim_per_band"] = per
                rep["ssim"] = float(per.mean())
            out.append(rep)
        return out


def decode_eval(enc: Encoded, orig=None, frames: torch.Tensor | None = None, want_ssim: bool = True,
                want_recon: bool = True, recon_out: torch.Tensor | None = None):
    """Frames (the codec's decoded output; default: ``enc.frames``) -> recon + scores.

    Scores are taken against the forward-filled original:
    ``enc.filled`` when the encoder produced it, else ``orig``.
    """
    B, T, H, W, C = enc.shape
    ref = enc.filled if enc.filled is not None else orig
    if ref is None:
        raise ConfigurationError("decode_eval needs the original cube to score against")
    o, shp = _as_batch(ref)
    if shp != enc.shape:
        raise ConfigurationError(f"original {shp} does not match the encoded stream {enc.shape}")
    if want_ssim and (H < SSIM_WINDOW or W < SSIM_WINDOW):
        raise ConfigurationError(f"spatial dims {H}x{W} smaller than the {SSIM_WINDOW}-px SSIM window")
    fr = enc.frames if frames is None else frames
    if tuple(fr.shape) != tuple(enc.frames.shape):
        # a decoder handed back a different byte count: per video it must be a whole
        # number of HxWx3 frames (bridge.py:163-171), and as many frames as were encoded
        if fr.dtype != enc.frames.dtype:
            raise ConfigurationError(f"decoded frames are {fr.dtype}, the stream is {enc.frames.dtype}")
        n_videos = B * len(enc.groups)
        n_bytes = fr.numel() * fr.element_size()
        per_video = n_bytes // n_videos if n_bytes % n_videos == 0 else n_bytes
        got = check_stream_bytes(per_video, H, W, 3, enc.spec.bit_depth)
        if n_bytes % n_videos != 0 or got != T:
            raise CorruptStreamError(f"decoded {got} frames per video, the stream holds {T}")
        fr = fr.contiguous().view(enc.frames.shape)
    d = o.device
    s = dev.stream_ptr(d)
    lib = _lib.load()
    E = enc.n_encoded
    recon = None
    if want_recon:
        recon = recon_out if recon_out is not None else torch.empty(
            (B, T, H, W, C) if len(o.shape) == 5 else (T, H, W, C), dtype=torch.float32, device=d)
    sse = torch.empty((B, C), dtype=torch.float64, device=d)
    ssum = torch.zeros((B, C), dtype=torch.float64, device=d)
    ws = dev.workspace(lib.cv_eval_ws_bytes(B, T, H, W, C, int(want_ssim)), d)
    err = enc.err if enc.err is not None else dev.ErrWord(d)
    fdt = _lib.CV_U8 if fr.dtype == torch.uint8 else _lib.CV_U16
    if not enc.pca:
        _lib.call("cv_eval", fr.data_ptr(), fdt, E, enc.qmins.data_ptr(), enc.qmaxs.data_ptr(),
                  enc.spec.bit_depth, None, None, None, 0, o.ptr, o.code, B, T, H, W, C,
                  enc.peaks.data_ptr(), int(want_ssim), recon.data_ptr() if recon is not None else None,
                  ws.data_ptr(), sse.data_ptr(), ssum.data_ptr(), err.ptr, s)
    else:
        for b in range(B):
            fold = enc.pca[b]
            o_b = o.t[b] if o.t.dim() == 5 else o.t
            r_b = None
            if recon is not None:
                r_b = (recon[b] if recon.dim() == 5 else recon).data_ptr()
            _lib.call("cv_eval", fr[b].data_ptr(), fdt, E, enc.qmins[b:].data_ptr(),
                      enc.qmaxs[b:].data_ptr(), enc.spec.bit_depth, fold.inv_mean.ctypes.data,
                      fold.inv_comps.ctypes.data, None, 0, o_b.data_ptr(), o.code, 1, T, H, W, C,
                      enc.peaks[b:].data_ptr(), int(want_ssim), r_b, ws.data_ptr(),
                      sse[b:].data_ptr(), ssum[b:].data_ptr(), err.ptr, s)
    Tg = T
    if enc.shard is not None and enc.t_total is not None:
        sse, ssum = enc.shard.combine_scores(sse, ssum)  # per-band partial sums of all time shards
        Tg = enc.t_total
    scores = Scores(sse, ssum, enc.peaks, Tg * H * W,
                    Tg * (H - SSIM_WINDOW + 1) * (W - SSIM_WINDOW + 1) if want_ssim else 0,
                    want_ssim, enc.frame_bytes // B * Tg // T, (B, Tg, H, W, C))
    return recon, scores


def roundtrip(cube, spec: StreamSpec, want_ssim: bool = True, want_recon: bool = True):
    """encode_prep -> (identity codec) -> decode_eval; returns (encoded, recon, scores)."""
    if not dev.is_device_tensor(cube):
        cube = dev.to_device(cube).t
    enc = encode_prep(cube, spec)
    recon, scores = decode_eval(enc, cube, want_ssim=want_ssim, want_recon=want_recon)
    return enc, recon, scores


class HostStreamer:
    """End-to-end round trips of host-resident cubes through the public API,
    including the codec hand-off on both sides (SPEC.md:351/360,
    bridge.py:157-160, 213-230, 288-303).

    Per chunk of cubes: the cube is copied from pinned host memory (H2D copy
    stream) -> ``encode_prep`` -> every ``[b][g]`` frame slice (the bytes
    ``_frames_to_planar_bytes`` hands ffmpeg for video g) is copied into
    pinned host frames, one ``cudaMemcpyAsync`` per slice (D2H copy stream)
    -> the codec's decoded frames are copied back (H2D; the benchmark's codec
    is the identity, so they are the same bytes) -> ``decode_eval`` scores them
    -> the per-band metric sums come back to the host. With more than one
    chunk the copies of one chunk overlap the kernels of the other (two
    buffer sets). ``shard`` (dist.TimeShard) runs a time-sharded stream.
    """

    def __init__(self, shape, dtype, spec: StreamSpec, chunk: int, want_ssim: bool = True,
                 device=None, handoff: bool = True, shard=None):
        self.B, self.T, self.H, self.W, self.C = shape
        self.spec = spec
        self.chunk = max(1, min(chunk, self.B))
        self.want_ssim = want_ssim
        self.handoff = handoff
        self.shard = shard
        self.device = device or dev.default_device()
        nchunks = (self.B + self.chunk - 1) // self.chunk
        self.nbuf = 2 if nchunks > 1 else 1
        per = (self.chunk, self.T, self.H, self.W, self.C)
        self.bufs = [torch.empty(per, dtype=dtype, device=self.device) for _ in range(self.nbuf)]
        self.recon = torch.empty(per, dtype=torch.float32, device=self.device)
        self.h2d_stream = torch.cuda.Stream(self.device)
        self.d2h_stream = torch.cuda.Stream(self.device)
        self.ready = [torch.cuda.Event() for _ in range(self.nbuf)]
        self.free = [torch.cuda.Event() for _ in range(self.nbuf)]
        self.ws = [Workspace() for _ in range(self.nbuf)]
        E = spec.n_pcs or self.C
        G = (E + 2) // 3
        tdt, _ = dev.out_dtype_for_depth(spec.bit_depth)
        fshape = (self.chunk, G, self.T, 3, self.H * self.W)
        self.host_frames = None
        if handoff:
            self.host_frames = [torch.empty(fshape, dtype=tdt, pin_memory=True) for _ in range(self.nbuf)]
            self.dec = [torch.empty(fshape, dtype=tdt, device=self.device) for _ in range(self.nbuf)]
        self.h2d_bytes = 0
        self.d2h_bytes = 0

    def run(self, host: torch.Tensor) -> list:
        """host: pinned [B,T,H,W,C]; returns one metric report per cube."""
        comp = torch.cuda.current_stream(self.device)
        sse, ssim, peaks = [], [], []
        starts = list(range(0, self.B, self.chunk))
        self.h2d_bytes = 0
        self.d2h_bytes = 0

        def issue(i):
            k = i % self.nbuf
            s0 = starts[i]
            n = min(self.chunk, self.B - s0)
            with torch.cuda.stream(self.h2d_stream):
                self.h2d_stream.wait_event(self.free[k])
                self.bufs[k][:n].copy_(host[s0:s0 + n], non_blocking=True)
                self.ready[k].record(self.h2d_stream)
            self.h2d_bytes += host[s0:s0 + n].numel() * host.element_size()

        for k in range(self.nbuf):
            self.free[k].record(comp)
        issue(0)
        scores = None
        for i, s0 in enumerate(starts):
            k = i % self.nbuf
            n = min(self.chunk, self.B - s0)
            if i + 1 < len(starts) and self.nbuf > 1:
                issue(i + 1)
            comp.wait_event(self.ready[k])
            x = self.bufs[k][:n]
            enc = encode_prep(x, self.spec, workspace=self.ws[k], shard=self.shard)
            frames = None
            if self.handoff:
                frames = self._handoff(enc, k, n, comp)
            _, scores = decode_eval(enc, x, frames=frames, want_ssim=self.want_ssim,
                                    recon_out=self.recon[:n])
            self.free[k].record(comp)
            if i + 1 < len(starts) and self.nbuf == 1:
                issue(i + 1)
            sse.append(scores.sse)
            ssim.append(scores.ssim_sum)
            peaks.append(scores.peaks)
        allsse = torch.cat(sse).cpu()
        allssim = torch.cat(ssim).cpu()
        allpeaks = torch.cat(peaks).cpu()
        self.d2h_bytes += 3 * allsse.numel() * 8
        out = Scores(allsse, allssim, allpeaks, scores.n_per_band, scores.n_ssim_per_band,
                     self.want_ssim, scores.frame_bytes_per_cube, (self.B,) + tuple(scores.shape[1:]))
        return out.report()

    def _handoff(self, enc: Encoded, k: int, n: int, comp) -> torch.Tensor:
        """Frames -> pinned host (one copy per [b][g] video slice) -> decoded frames -> device."""
        hf = self.host_frames[k][:n]
        dec = self.dec[k][:n]
        done = torch.cuda.Event()
        done.record(comp)
        self.d2h_stream.wait_event(done)
        arrived = None
        # one video slice at a time: the slice goes to the host (where the codec runs), and its
        # decoded frames come back while the next slice is still on its way out (PCIe is full duplex)
        for b in range(n):
            for g in range(enc.frames.shape[1]):
                with torch.cuda.stream(self.d2h_stream):
                    hf[b, g].copy_(enc.frames[b, g], non_blocking=True)
                    back = torch.cuda.Event()
                    back.record(self.d2h_stream)
                with torch.cuda.stream(self.h2d_stream):
                    self.h2d_stream.wait_event(back)
                    dec[b, g].copy_(hf[b, g], non_blocking=True)
                    arrived = torch.cuda.Event()
                    arrived.record(self.h2d_stream)
        nbytes = hf.numel() * hf.element_size()
        self.d2h_bytes += nbytes
        self.h2d_bytes += nbytes
        comp.wait_event(arrived)
        return dec
