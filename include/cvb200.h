/*
 * cvb200.h — C ABI of the B200 (sm_100a) array-side hot path of the cubevid /
 * xarrayvideo pipeline ("Video Compression for Spatiotemporal Earth System
 * Data", arXiv 2506.19656).
 *
 * The reference (`/root/reference/pkg/src/cubevid`) is a pure-numpy Python
 * package: its hot path is a set of plain Python functions on numpy arrays,
 * with no FFI. This header is the boundary the Python drop-in
 * (`paper_2506_19656_b200`) binds with ctypes; every entry point names the
 * reference function(s) it replaces.
 *
 * Conventions
 *  - All array pointers are DEVICE pointers owned by the caller; the library
 *    never allocates or frees caller memory and keeps no global state except a
 *    per-thread last-error string.
 *  - `stream` is a `cudaStream_t` passed as `void*` (NULL = legacy stream).
 *    No entry point synchronises the host; device-side error conditions are
 *    OR-ed into the caller's `uint32_t* err_word` (device memory, CV_FLAG_*),
 *    which the caller reads once per call (or once per pipeline step).
 *  - Cubes are channel-last `[n_cubes][T][H*W][C]` (transform.py:62,
 *    cube.py:250). Video frames are planar `[n_cubes][G][T][3][H*W]`, G =
 *    ceil(E/3) groups of three planes, little-endian u8 (B=8) or u16 (B>8)
 *    (bridge.py:157-160, plan.py:118-128).
 *  - Return value: CV_OK or a CV_ERR_* status (argument/shape errors are
 *    detected on the host before any launch).
 */
#ifndef CVB200_H
#define CVB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (host-side validation) -> ConfigurationError in Python */
enum {
  CV_OK = 0,
  CV_ERR_ARG = 1,         /* bad argument value (bit depth, dtype, null pointer) */
  CV_ERR_SHAPE = 2,       /* inconsistent sizes */
  CV_ERR_UNSUPPORTED = 3, /* valid for the reference, not supported by this build */
  CV_ERR_CUDA = 4         /* a CUDA launch failed */
};

/* device error-word flags (atomicOr'ed by kernels) */
enum {
  CV_FLAG_NONFINITE = 1u, /* +/-inf in float input (cube.py:229-230, transform.py:66-67) */
  CV_FLAG_NAN = 2u,       /* NaN where no fill policy applies (transform.py:66-67)       */
  CV_FLAG_RANGE = 4u,     /* value outside [min,max] without clamp (transform.py:94-97)  */
  CV_FLAG_INT_RANGE = 8u  /* integer sample > 2^B-1 (transform.py:115-119)              */
};

/* element types */
enum { CV_U8 = 0, CV_U16 = 1, CV_F32 = 2, CV_F64 = 3 };

/* frame layouts */
enum { CV_LAYOUT_CHANNEL_LAST = 0, CV_LAYOUT_PLANAR = 1 };
/* padding of the last 3-plane group: repeat last real channel (plan.py:126) or zeros */
enum { CV_PAD_REPEAT = 0, CV_PAD_ZERO = 1 };

/* version = 10000*major + 100*minor + patch */
int cv_version(void);
const char *cv_status_string(int status);
/* message of the last failing call on this host thread ("" if none) */
const char *cv_last_error(void);
/* largest channel count the kernels accept (per stream) */
int cv_max_channels(void);
/* number of kernels this library has launched in the process (benchmark accounting) */
unsigned long long cv_launch_count(void);
/* Select a kernel variant for A/B measurements and tests (process-wide; set it
 * before launching, not concurrently with launches). Names: "gram_tiles" (0/1),
 * "gram_nt" (64 or 256), "gram_checks" (0/1), "gram12" (0/1), "proj_nopf" (0/1), "proj12" (0/1), "qp_px1" (0/1),
 * "qp_runtime_c" (0/1),
 * "eval_kernel" (0 / 8 = k_eval_ssim8, the default; 7 = k_eval_ssim7).
 * Defaults are the measured-fastest variants. Unknown names / values: CV_ERR_ARG. */
int cv_set_variant(const char *name, int value);

/* ---------------------------------------------------------------------- */
/* K1 — per-band statistics (+ forward-fill segment carries)               */
/* ---------------------------------------------------------------------- */

/* bytes of the statistics workspace for n_cubes x C bands */
size_t cv_stats_ws_bytes(int64_t n_cubes, int32_t C);
/* number of time segments of length seg_len (carry map has n_seg*inner floats per cube) */
int64_t cv_num_segments(int64_t T, int32_t seg_len);

/*
 * Reset a statistics workspace (must precede cv_stats).
 */
int cv_stats_reset(void *stats_ws, int64_t n_cubes, int32_t C, void *stream);

/*
 * Replaces fit_quant's observation pass (transform.py:61-70) and the NaN scan
 * of forward_fill_time (cube.py:229-238).
 * src: [n_cubes][T][inner] of `dtype`; band of an element = (index in inner) % C.
 * fill_mode 0: NaN is an error (CV_FLAG_NAN), as in fit_quant.
 * fill_mode 1: NaN cells are forward-filled along T; min/max run over the
 *              observed values plus the leading-fill constant when any
 *              t=0 cell of the band is NaN. If seg_last != NULL it receives,
 *              per segment of seg_len steps, the last observed value of each
 *              element (NaN if none): [n_cubes][n_seg][inner] f32.
 * +/-inf always sets CV_FLAG_NONFINITE.
 */
int cv_stats(const void *src, int32_t dtype, int64_t n_cubes, int64_t T,
             int64_t inner, int32_t C, int32_t fill_mode, int32_t seg_len,
             void *stats_ws, float *seg_last, uint32_t *err_word, void *stream);

/*
 * Turn a statistics workspace into fit_quant's float64 ranges
 * (transform.py:68-70): mins/maxs [n_cubes][C]; nan_counts (nullable)
 * [n_cubes][C] = ValidityMask.n_synthesized per band (cube.py:43-45).
 */
int cv_stats_finalize(const void *stats_ws, int64_t n_cubes, int32_t C,
                      int32_t fill_mode, float fill_value, double *mins,
                      double *maxs, int64_t *nan_counts, void *stream);

/*
 * Per (cube, band) leading-gap flag of a fill-mode statistics workspace
 * (1 = some t=0 cell of the band was NaN, so the leading fill constant enters
 * the band's range, cube.py:236-242): lead [n_cubes][C] int32. Time-sharded
 * streams combine the flag of the first shard only (dist.py).
 */
int cv_stats_lead_flags(const void *stats_ws, int64_t n_cubes, int32_t C,
                        int32_t *lead, void *stream);

/* ---------------------------------------------------------------------- */
/* forward_fill_time (cube.py:213-246)                                      */
/* ---------------------------------------------------------------------- */

/*
 * src/out: [n_outer][T][inner] f32 (time axis moved to position 1 by the
 * caller's strides); mask (nullable): same shape, 1 = observed (ValidityMask).
 * seg_last: carry map produced by cv_stats(fill_mode=1, seg_len) over the
 * same geometry (C = 1 is fine). carry_in (nullable, [n_outer][inner], NaN =
 * none): values carried in from earlier time shards (multi-GPU T-sharding).
 * Leading gaps take (float)fill_value.
 */
int cv_forward_fill(const float *src, int64_t n_outer, int64_t T, int64_t inner,
                    float fill_value, int32_t seg_len, const float *seg_last,
                    const float *carry_in, float *out, uint8_t *mask,
                    uint32_t *err_word, void *stream);

/* ---------------------------------------------------------------------- */
/* K4 — quantisation into integer frames                                   */
/* ---------------------------------------------------------------------- */

/*
 * Bit-exact replacement of quantize (transform.py:77-105): per element
 * q = floor(((v - min)/span)*(2^B-1) + 0.5) evaluated as the reference does in
 * IEEE float64 (constant channels -> 0), optional clamp (transform.py:92-93).
 *
 * src: [n_cubes][T][HW][C] (dtype). E = encoded channels = C, or n_pcs when
 * pca_comps != NULL: then each pixel is first projected,
 * pc_j = sum_c (v_c - pca_mean_c) * pca_comps[j][c] in float64
 * (transform.py:199). pca_mean [C] and pca_comps [n_pcs][C] are HOST
 * pointers (the model comes from the host eigh); they are passed to the
 * kernel by value and shared by all n_cubes.
 * mins/maxs: [n_cubes][E] float64.
 * fill_mode 1 forward-fills NaN along T using seg_last (see cv_stats) and
 * carry_in (nullable [n_cubes][HW*C]: carries from earlier time shards);
 * filled_out (nullable, f32 input only) then receives the filled cube, i.e.
 * forward_fill_time's output (cube.py:244-246), in the same pass.
 * out_layout CHANNEL_LAST: out [n_cubes][T][HW][E] (what quantize returns).
 * out_layout PLANAR: out [n_cubes][G][T][3][HW], planes padded per pad_mode
 *   (plan.py:118-128 + bridge.py:157-160).
 * Output type is u8 for bit_depth 8, u16 otherwise (transform.py:73-74).
 */
int cv_quantize(const void *src, int32_t dtype, int64_t n_cubes, int64_t T,
                int64_t HW, int32_t C, const double *mins, const double *maxs,
                int32_t bit_depth, int32_t clamp, int32_t fill_mode,
                float fill_value, int32_t seg_len, const float *seg_last,
                const float *carry_in, const double *pca_mean,
                const double *pca_comps, int32_t n_pcs,
                int32_t out_layout, int32_t pad_mode, void *out,
                float *filled_out, uint32_t *err_word, void *stream);

/*
 * dequantize (transform.py:108-126), bit-exact in float64:
 * out = min + (q / (2^B-1)) * (max - min); constant channels -> min.
 * q: channel-last [n][T][HW][E] or planar [n][G][T][3][HW] (padded planes
 * skipped). out: channel-last [n][T][HW][E], f32 (rounded once) or f64.
 * q > 2^B-1 sets CV_FLAG_INT_RANGE.
 */
int cv_dequantize(const void *q, int32_t qdtype, int64_t n_cubes, int64_t T,
                  int64_t HW, int32_t E, int32_t in_layout, const double *mins,
                  const double *maxs, int32_t bit_depth, void *out,
                  int32_t out_dtype, uint32_t *err_word, void *stream);

/* ---------------------------------------------------------------------- */
/* K2/K3 — band PCA                                                        */
/* ---------------------------------------------------------------------- */

size_t cv_gram_ws_bytes(int64_t n_pix, int32_t C);
/*
 * One-pass float64 shifted Gram over n_pix pixel spectra (transform.py:172-179):
 * out[0:C] = sum_p (x_p - s), out[C:C+C*C] = sum_p (x_p - s)(x_p - s)^T with
 * the shift s = the first pixel's spectrum (a device-side read; keeps the
 * one-pass sums well conditioned). Deterministic (fixed reduction tree).
 * src [n_pix][C] of dtype. stats_ws (nullable) also receives the per-band
 * min/max of the same pass (reset it first). Non-finite input sets
 * CV_FLAG_NONFINITE / CV_FLAG_NAN.
 */
int cv_pca_gram(const void *src, int32_t dtype, int64_t n_pix, int32_t C,
                void *ws, double *out, void *stats_ws, uint32_t *err_word,
                void *stream);

/*
 * pca_forward (transform.py:191-199) in float64 + per-component min/max
 * (fit_quant on the components). mean [C] / comps [K][C] are
 * HOST pointers (passed by value):
 * out (nullable) [n_cubes][n_pix][K] f32/f64; stats_ws (nullable) receives the
 * component ranges (finalize with cv_stats_finalize(C=K, fill_mode=0)).
 */
int cv_pca_project(const void *src, int32_t dtype, int64_t n_cubes,
                   int64_t n_pix, int32_t C, const double *mean,
                   const double *comps, int32_t K, void *out,
                   int32_t out_dtype, void *stats_ws, uint32_t *err_word,
                   void *stream);

/*
 * pca_inverse (transform.py:202-210): out = pc @ comps + mean, float64 math;
 * mean [C] / comps [K][C] are HOST pointers.
 * pc [n_cubes][n_pix][K] f32/f64 -> out [n_cubes][n_pix][C] f32/f64.
 */
int cv_pca_inverse(const void *pc, int32_t dtype, int64_t n_cubes,
                   int64_t n_pix, int32_t K, const double *mean,
                   const double *comps, int32_t C, void *out,
                   int32_t out_dtype, void *stream);

/* ---------------------------------------------------------------------- */
/* K5+K6 — decode + fidelity metrics                 */
/* ---------------------------------------------------------------------- */

size_t cv_eval_ws_bytes(int64_t n_cubes, int64_t T, int64_t H, int64_t W,
                        int32_t C, int32_t want_ssim);

/*
 * Reconstruct and score in one pass.
 * Reconstruction source, exactly one of:
 *   frames   planar [n][G][T][3][HW] (fdtype u8/u16), E encoded channels,
 *            dequantised with qmins/qmaxs [n][E] at bit_depth, then, when
 *            inv_comps != NULL, inverse-projected: x_c = sum_j pc_j *
 *            inv_comps[j][c] + inv_mean[c] (HOST pointers [E][C], [C],
 *            shared by all cubes, passed by value);
 *   recon_in channel-last [n][T][HW][C] (rdtype f32/f64).
 * Original: orig [n][T][HW][C] (odtype f32/f64/u16), already forward-filled
 * (the codec saw the filled cube): pass cv_quantize's
 * filled_out or cv_forward_fill's output. NaN sets CV_FLAG_NAN.
 * Outputs: recon_out (nullable) channel-last f32; sse [n][C] = sum of squared
 * error in float64; when want_ssim, ssim_sum [n][C] = sum over the valid
 * (H-10)x(W-10) region of every frame of the 11x11 Gaussian (sigma 1.5)
 * SSIM map with K1=0.01, K2=0.03 and dynamic range peaks[n][C].
 */
int cv_eval(const void *frames, int32_t fdtype, int32_t E, const double *qmins,
            const double *qmaxs, int32_t bit_depth, const double *inv_mean,
            const double *inv_comps, const void *recon_in, int32_t rdtype,
            const void *orig, int32_t odtype, int64_t n_cubes, int64_t T,
            int64_t H, int64_t W, int32_t C, const double *peaks,
            int32_t want_ssim, float *recon_out, void *ws, double *sse,
            double *ssim_sum, uint32_t *err_word, void *stream);

/* ---------------------------------------------------------------------- */
/* layout: select_for_video (cube.py:249-305), planar bytes (bridge.py:157-174) */
/* ---------------------------------------------------------------------- */

/*
 * select_for_video (cube.py:249-305): stack C channels into a contiguous
 * channel-last out [T][H][W][C]. chan_ptrs: HOST array of C DEVICE pointers,
 * channel c of the result (a 3-D variable, or one index of a 4-D variable's
 * channel axis). strides: HOST array [C][3], element strides of channel c
 * along the (t, y, x) roles of axis_order (the transposition the reference does
 * with np.transpose). Elements are moved as raw words of elem_size bytes
 * (1, 2, 4 or 8); all channels share the element type.
 */
int cv_select_stack(const void *const *chan_ptrs, const int64_t *strides,
                    int32_t C, int32_t elem_size, int64_t T, int64_t H,
                    int64_t W, void *out, void *stream);

/*
 * _frames_to_planar_bytes (bridge.py:157-160): q channel-last [T][HW][n_planes]
 * (u8/u16) -> out planar [T][n_planes][HW], the byte stream one video's
 * encoder reads (little-endian u16 is the device's native order).
 */
int cv_planar_pack(const void *q, int32_t dtype, int64_t T, int64_t HW,
                   int32_t n_planes, void *out, void *stream);

/*
 * _planar_bytes_to_frames (bridge.py:163-174): planes [T][n_planes][HW] ->
 * out channel-last [T][HW][n_planes]. The whole-frames byte-count check
 * (CorruptStreamError, bridge.py:167-171) is the caller's (host arithmetic).
 */
int cv_planar_unpack(const void *planes, int32_t dtype, int64_t T, int64_t HW,
                     int32_t n_planes, void *out, void *stream);

/* ---------------------------------------------------------------------- */
/* spectral angle                           */
/* ---------------------------------------------------------------------- */

size_t cv_angle_ws_bytes(void);
/*
 * Per pixel theta = arccos(<o, r> / (|o| |r|)) over the C channels (float64),
 * orig/recon channel-last [n_pix][C]. out (device, 3 doubles): sum of theta in
 * degrees over pixels with non-zero norms, their count, the skipped count.
 */
int cv_spectral_angle(const void *orig, int32_t odtype, const void *recon,
                      int32_t rdtype, int64_t n_pix, int32_t C, void *ws,
                      double *out, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* CVB200_H */
