/*
 * infigrid_b200 — C-ABI of the B200-native InfiniteDiffusion sampling hot path.
 *
 * Plain pointers and sizes only (no torch types).  Every data pointer is a
 * DEVICE pointer owned by the caller; `stream` is a cudaStream_t (may be 0).
 * Functions return 0 (IG_OK) or an IG_ERR_* code; ig_last_error() returns a
 * thread-local message for the last failure.  Integer lattice coordinates are
 * int64 and follow Python floor-division semantics, as the reference does.
 *
 * Reference interfaces replaced (all paths under /root/reference/pkg/src/infigrid/):
 *   ig_noise_region        noise.py:74-86   noise_region / noise_at (:67-71)
 *   ig_phi_analytic        denoise.py:89-113 apply (identity/shrink_smooth/cond_affine;
 *                          multistep = repeated calls), box_mean transforms.py:29-51,
 *                          conditioning fill denoise.py:116-163
 *   ig_blend               store.py:428-436 _accumulate (+ sampler.py:151-154 W*Phi
 *                          contribution) and store.py:549-554 divide_weighted
 *   ig_box_mean            transforms.py:29-51
 *   ig_blur_block_mean_f64 transforms.py:54-67 (block_mean of blur3_iterated, float64)
 *   ig_block_mean          transforms.py:61-67 block_mean (float32 / float64 accumulation)
 *   ig_upsample_nn         transforms.py:70-72 upsample_nn
 *   ig_normalize_u8        transforms.py:117-135 normalize_heightmap_u8 (render path)
 *   ig_hillshade_u8        cli.py:230-249 hillshade (render --hillshade)
 *   ig_convert             numpy astype at transforms.py:93,101 (dtype-preserving decode)
 *   ig_laplacian_residual  transforms.py:89-95 (high = x - up(low))
 *   ig_laplacian_merge     transforms.py:98-101 / :104-114 (up(low)+high [, signed_square])
 *   ig_signed_pow          transforms.py:17-26
 *   ig_patch_features      denoise.py:166-185 coarse_patch_features
 *   ig_condition_window    denoise.py:116-163 conditioning_for_window (batched)
 *   ig_procedural_map      pipeline.py:101-123 ProceduralMap.values
 *   ig_corrupt             pipeline.py:126-139 corrupt_user_map
 *   ig_raster_map          pipeline.py:72-84 RasterMap.values
 *   ig_pack_windows / ig_ipc_event_*   the halo exchange of the sharded query
 *                          (no reference counterpart: the reference is
 *                          single-process)
 *   ig_tiles_resolve       store.py:364-426 _gather_tiles + _commit_region of
 *                          _read_indirect (INDIRECT tile cache in HBM)
 *   ig_unet_*              the Phi plugin (denoise.py:89 apply) for the new "unet" kind;
 *                          no reference implementation exists
 */
#ifndef INFIGRID_B200_H
#define INFIGRID_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IG_OK 0
#define IG_ERR_ARG 1          /* bad shape/argument  -> ShapeError / ValueError   */
#define IG_ERR_CUDA 2         /* CUDA runtime error  -> StoreError              */
#define IG_ERR_UNSUPPORTED 3  /* unsupported config  -> ConfigError             */

#define IG_DTYPE_F32 0
#define IG_DTYPE_F64 1
#define IG_DTYPE_F16 2   /* storage-only types of the dtype-generic transforms */
#define IG_DTYPE_I32 3
#define IG_DTYPE_I64 4

#define IG_PHI_IDENTITY 0
#define IG_PHI_SHRINK_SMOOTH 1
#define IG_PHI_COND_AFFINE 2

const char* ig_last_error(void);
int ig_abi_version(void);
/* number of kernels this library has launched in the process (instrumentation) */
long long ig_launch_count(void);

/* ---- K1 noise ----------------------------------------------------------
 * out[(c*height + py)*width + px] = G(seed, stream, x0+px, y0+py, ch0+c),
 * float32 (or its exact float64 widening when out_dtype == IG_DTYPE_F64).
 * slow_count (nullable, device int32): incremented once per CTA that took the
 * exact double-double path (diagnostic). */
int ig_noise_region(uint64_t seed, uint32_t stream, int64_t x0, int64_t y0,
                    int32_t width, int32_t height, int32_t ch0, int32_t nch,
                    int32_t out_dtype, void* out, int32_t* slow_count, void* cuda_stream);

/* ---- K3 analytic Phi over a batch of square windows ---------------------
 * Window k covers [wxy[2k], +window) x [wxy[2k+1], +window) on the lattice.
 * Source: if src_batched, src is [n][channels][window][window]; otherwise a
 * canvas (channels, src_h, src_w) whose pixel (0,0) sits at (src_x0, src_y0).
 * Output: out[n][channels][window][window] (dtype = dtype of src).
 * Conditioning (cond_affine): cond_parent is (cond_c, cond_h, cond_w) on a
 * lattice `cond_scale` times coarser, origin (cond_x0, cond_y0); NULL means
 * y = None.  cond_mask_channel < 0 means an all-ones mask.  Holes (mask < 1)
 * read noise stream 101 of cond_seed when cond_fill != 0 (cond_fill == 0: the
 * parent's channel 0 is used as is -- a materialised Conditioning). */
int ig_phi_analytic(int32_t kind, int32_t radius, double lam, int32_t dtype,
                    const void* src, int32_t src_batched, int64_t src_x0, int64_t src_y0,
                    int32_t src_w, int32_t src_h, int32_t channels,
                    const int64_t* wxy, int32_t n, int32_t window,
                    const void* cond_parent, int64_t cond_x0, int64_t cond_y0,
                    int32_t cond_w, int32_t cond_h, int32_t cond_c, int32_t cond_scale,
                    int32_t cond_mask_channel, uint64_t cond_seed, int32_t cond_fill,
                    void* out, void* cuda_stream);

/* ---- K5 canonical-order blend -------------------------------------------
 * win_data: device array of nj*ni pointers, entry (j-j0)*ni + (i-i0) is the
 * stored data of window (i, j) or NULL (skipped).  mode 0: entries hold full
 * contributions with `channels` channels, summed as stored.  mode 1: entries
 * hold Phi outputs with `channels` data channels; the contribution is
 * fl(W*Phi) plus a weight channel W (W = window x window table, `weight`).
 * Output (region rw x rh at (rx0, ry0)):
 *   divide == 0: raw sums, mode 0 -> channels planes, mode 1 -> channels+1
 *   divide == 1: (mode 1 only) data / weight where weight > 0 else 0. */
int ig_blend(const void* const* win_data, int64_t i0, int64_t j0, int32_t ni, int32_t nj,
             int32_t window, int32_t stride, int64_t off_x, int64_t off_y,
             int32_t channels, int32_t mode, const void* weight,
             int64_t rx0, int64_t ry0, int32_t rw, int32_t rh,
             int32_t divide, int32_t dtype, void* out, void* cuda_stream);

/* weighted read over a region (divide_weighted on raw (C+1) planes) */
int ig_divide_weighted(const void* raw, int32_t channels, int64_t npix, int32_t dtype,
                       void* out, void* cuda_stream);

/* ---- peer-memory halo exchange (cfg5 sharding) -------------------
 * Replaces the send/recv of boundary Phi windows (shard.py p2p_exchange) by
 * mapping the producer's allocation: export on the producer, open on the
 * consumer (peer access enabled lazily from the consumer's current device), and
 * the consumer's ig_blend reads the windows in place over NVLink.
 * handle64: 64-byte cudaIpcMemHandle_t of the allocation containing dev_ptr;
 * offset: dev_ptr - allocation base.  ig_ipc_open returns the mapped base. */
int ig_ipc_export(const void* dev_ptr, uint8_t* handle64, int64_t* offset);
int ig_ipc_open(const uint8_t* handle64, void** base_out);
int ig_ipc_close(void* base);
/* dedicated exchange buffer (plain cudaMalloc, outside torch's caching pool, so
 * a peer maps only the exchanged windows) */
int ig_ipc_alloc(int64_t bytes, void** ptr_out);
int ig_ipc_free(void* ptr);
/* one launch copies n windows (window_bytes each, a multiple of 16) from the
 * device addresses src_ptrs[k] (a device table) into consecutive slots of dst:
 * the producer's pack of its outgoing boundary windows */
int ig_pack_windows(const int64_t* src_ptrs, int32_t n, int64_t window_bytes, void* dst,
                    void* cuda_stream);
/* cross-process device ordering of the exchange: the producer records an
 * interprocess event after its pack, the consumer's stream waits on it before
 * the blends that read the windows (64-byte cudaIpcEventHandle_t) */
int ig_ipc_event_create(uint8_t* handle64, void** event_out);
int ig_ipc_event_open(const uint8_t* handle64, void** event_out);
int ig_event_record(void* event, void* cuda_stream);
int ig_stream_wait_event(void* cuda_stream, void* event);
int ig_event_destroy(void* event);

/* ---- INDIRECT tile cache (store.py:358-426) ---------------------------------
 * table[2*(ty*ntx + tx)] = device pointer of tile (tx0+tx, ty0+ty)'s data
 * (channels, tile_size, tile_size), table[... + 1] its finalized mask
 * (tile_size^2 bytes, 0/1).  Every tile of the box that the region touches must
 * exist.  Per pixel of the region (origin rx0, ry0; out is (channels, rh, rw)):
 * finalized -> out = tile value; otherwise tile = out and the pixel becomes
 * finalized (the reference's gather of finalized pixels followed by the commit
 * of the whole region, in one pass).  elem_bytes 4 (float32) or 8 (float64). */
int ig_tiles_resolve(const int64_t* table, int64_t tx0, int64_t ty0, int32_t ntx, int32_t nty,
                     int32_t tile_size, int32_t channels, int32_t elem_bytes, int64_t rx0,
                     int64_t ry0, int32_t rw, int32_t rh, void* out, void* cuda_stream);

/* ---- K6 elevation transforms ---------------------------------------------- */
int ig_box_mean(const void* in, int32_t planes, int32_t h, int32_t w, int32_t radius,
                int32_t dtype, void* out, void* cuda_stream);
/* low = block_mean(blur3_iterated(in, blur_iters), factor), all float64;
 * in_dtype selects the input element type (widened exactly). scratch: 2 planes*h*w f64 */
int ig_blur_block_mean_f64(const void* in, int32_t in_dtype, int32_t planes, int32_t h,
                           int32_t w, int32_t blur_iters, int32_t factor, double* scratch,
                           double* low, void* cuda_stream);
/* high = widen(x) - up(low) */
int ig_laplacian_residual(const void* x, int32_t x_dtype, const double* low, int32_t planes,
                          int32_t h, int32_t w, int32_t factor, double* high, void* cuda_stream);
/* out = cast(up(low) + high) [then signed_square in out dtype when square_out] ;
 * out_dtype F64 keeps the provisional sum (stabilize); F16/I32/I64 outputs
 * are laplacian_decode's astype(original dtype) (no square_out) */
int ig_laplacian_merge(const double* low, const double* high, int32_t planes, int32_t h,
                       int32_t w, int32_t factor, int32_t out_dtype, int32_t square_out,
                       void* out, void* cuda_stream);
/* op 0: signed_sqrt (F32/F64), 1: signed_square (F32/F64, or I32/I64 with
 * two's-complement wraparound like numpy's integer multiply) */
int ig_signed_pow(const void* in, int64_t n, int32_t op, int32_t dtype, void* out,
                  void* cuda_stream);
/* block_mean (transforms.py:61-67) in the accumulation dtype numpy's .mean
 * uses (F32 for float32/float16 input, F64 otherwise), numpy's order: for
 * each of the f block rows the pairwise sum of its f values, added in row
 * order, then one division by f*f */
int ig_block_mean(const void* in, int32_t dtype, int32_t planes, int32_t h, int32_t w,
                  int32_t factor, void* out, void* cuda_stream);
/* elementwise astype between IG_DTYPE_* codes (exact widenings; RN narrowings;
 * float -> int truncates) */
int ig_convert(const void* in, int32_t in_dtype, int64_t n, void* out, int32_t out_dtype,
               void* cuda_stream);
/* normalize_heightmap_u8 (transforms.py:117-135): in (images, hw) float32 or
 * float64, out (images, 3, hw) uint8; minmax: device scratch of 2*images u64 */
int ig_normalize_u8(const void* in, int32_t dtype, int32_t images, int64_t hw, void* minmax,
                    uint8_t* out, void* cuda_stream);
/* hillshade (cli.py:230-249): Horn 3x3 slope shading of one (h, w) float32 /
 * float64 raster to uint8, float64 arithmetic; cos_zenith / sin_zenith /
 * azimuth as the reference computes them on the host */
int ig_hillshade_u8(const void* elev, int32_t dtype, int32_t h, int32_t w, double cos_zenith,
                    double sin_zenith, double azimuth, uint8_t* out, void* cuda_stream);
/* upsample_nn (transforms.py:70-72): out[p][Y][X] = in[p][Y/f][X/f], any
 * element size (1/2/4/8 bytes) */
int ig_upsample_nn(const void* in, int32_t elem_bytes, int64_t planes, int32_t h, int32_t w,
                   int32_t factor, void* out, void* cuda_stream);

/* ---- K7/K8/K9 hierarchy helpers ----------------------------------------------
 * features over a batch of n elevation tiles [n][h][w] (channel 0 of each
 * parent slab, row stride `in_stride_tile` elements between tiles):
 * out[n][3][h/patch][w/patch] = (mean, p-th rank, 1) */
int ig_patch_features(const void* in, int64_t tile_stride, int32_t n, int32_t h, int32_t w,
                      int32_t patch, int32_t rank, int32_t dtype, void* out,
                      void* cuda_stream);
/* conditioning_for_window for a batch: out[n][cond_c][window][window] channels
 * and mask_out[n][window][window] (both dtype) */
int ig_condition_window(const void* parent, int64_t px0, int64_t py0, int32_t pw, int32_t ph,
                        int32_t pc, int32_t scale, int32_t mask_channel, uint64_t seed,
                        const int64_t* wxy, int32_t n, int32_t window, int32_t dtype,
                        void* out, void* mask_out, void* cuda_stream);
int ig_procedural_map(uint64_t seed, uint32_t stream, int32_t cell, int64_t x0, int64_t y0,
                      int32_t w, int32_t h, int32_t channels, float* out, void* cuda_stream);
/* out[c] = in[c] + f32(level[c]) * G(seed, 201+c, ., ., 0) (level 0 -> copy) */
int ig_corrupt(const float* in, const double* levels_host, int32_t channels, uint64_t seed,
               int64_t x0, int64_t y0, int32_t w, int32_t h, float* out, void* cuda_stream);
/* RasterMap.values: mode 0 clamp, 1 tile; raster (rc, rh, rw) f32 */
int ig_raster_map(const float* raster, int32_t rc, int32_t rh, int32_t rw, int32_t mode,
                  int64_t x0, int64_t y0, int32_t w, int32_t h, int32_t channels, float* out,
                  void* cuda_stream);

/* ---- K4 UNet Phi (tcgen05/TMEM implicit-GEMM convolutions) -------------------
 * Implicit-GEMM 3x3 (taps = 9) or 1x1 (taps = 1) convolution, NHWC bf16:
 *   out[p][co] = epilogue( sum_{tap, ci} act[p + tap][ci] * wgt[co][tap][ci] )
 * act_a: [n][h][w][ca] and optional act_b: [n][h][w][cb] (channel concat,
 * used by decoder skips); ca, cb multiples of 64; cout multiple of 16, <= 256.
 * Epilogue (per output channel co, fp32):
 *   y = acc * scale[co] + bias[co]
 *   if (res)   y = res_a * res[p][co] + res_b * y                (mp_sum)
 *   out0[p][co] = bf16(y)            (if out0)
 *   out1[p][co] = bf16(act_gain * silu(y))   (if out1)
 * workspace: >= ig_conv_workspace_bytes() bytes of device memory (TMA maps). */
typedef struct {
  int32_t n, h, w, ca, cb, cout, taps;
  const void* act_a;
  const void* act_b;
  const void* wgt;        /* [cout][taps][ca+cb] bf16, K-major */
  const float* scale;     /* [cout] */
  const float* bias;      /* [cout] */
  const void* res;        /* [n][h][w][cout] bf16 or NULL */
  float res_a, res_b, act_gain;
  void* out0;             /* bf16 or NULL */
  void* out1;             /* bf16 or NULL */
  /* fused 1x1 skip GEMM accumulated into the same fp32 accumulator before the
   * epilogue:  acc += sum_ci concat(skip_a, skip_b)[p][ci] * wskip[co][ci]
   * (csa, csb multiples of 64; csa = 0 disables it).  Replaces a separate skip
   * convolution + residual read for mp_sum blocks. */
  int32_t csa, csb;
  const void* skip_a;     /* [n][h][w][csa] bf16 */
  const void* skip_b;     /* [n][h][w][csb] bf16 or NULL */
  const void* wskip;      /* [cout][csa+csb] bf16 */
  /* up2 != 0: out0/out1 are [n][2h][2w][cout] and every result is written to
   * its 2x2 block (nearest-neighbour upsample fused into the epilogue) */
  int32_t up2;
  /* up_in bit 0: act_a is [n][h/2][w/2][ca] and is read 2x nearest-upsampled;
   * bit 1: the same for skip_a.  The upsample happens inside the TMA load
   * (a zero-stride replicate dimension in the tensor map), so the full-res
   * tensor is never written.  Tensor-core path: halo kernel only (w % 128 ==
   * 0, taps == 9), otherwise IG_ERR_UNSUPPORTED; ig_conv_simt: any shape. */
  int32_t up_in;
  /* gutter bit 0: act_a, act_b, skip_a, skip_b, res, out0 and out1 use the
   * gutter layout [n][h][w+2][c] (zero columns at x = -1 and x = w; widths
   * <= 64): every 3x3 tap is then a 1-D shift over the h*(w+2) positions of
   * an image, so narrow levels run the CTA-pair halo kernel with one 1-D
   * halo box per chunk; the outputs' gutter columns are written as zeros.
   * bit 1: the up_in (low-res) sources are in the gutter layout;
   * bit 2: the fused-pool outputs (pool0/pool1) are in the gutter layout. */
  int32_t gutter;
  /* pool0 / pool1 (or NULL): the 2x2 mean pool of out0 and its mp_silu,
   * [n][h/2][w/2][cout], written by the same epilogue (bit-identical to
   * ig_avgpool2_bf16 on out0); CTA-pair kernel only (3x3, w % 128 == 0,
   * cout 64 / 128, 2-D layout). */
  void* pool0;
  void* pool1;
  /* head_norm 1 / 2: out0 = head_scale * x / (1e-4 + ||x|| / 8) per 64-channel
   * head of the (scaled) accumulator, stored bf16 / f16 -- EDM2 attention q, k /
   * v -- instead of the plain epilogue (cout % 128 == 0, out0 only). */
  int32_t head_norm;
  float head_scale;
} ig_conv_params_t;
size_t ig_conv_workspace_bytes(void);
/* 0: automatic; 1: force the per-tap kernel; 2: halo kernel instead of the row ring */
int ig_conv_set_variant(int force_per_tap);
int ig_conv_tc(const ig_conv_params_t* p, void* workspace, void* cuda_stream);
/* The EDM2 attention block's q / k / v 1x1 projections in one launch: wgt =
 * [3 cout][ca] bf16 (rows q | k | v), out0 = q (head_scale applied), k_out, v_out
 * (v as f16); head_norm must be 1, cout 256, taps 1.  Same results as three
 * ig_conv_tc calls with head_norm 1 / 1 / 2 (bit-identical). */
int ig_conv_qkv(const ig_conv_params_t* p, void* k_out, void* v_out, void* cuda_stream);
/* UNet helpers (NHWC bf16 activations):
 * ig_unet_gather_input: tap-packed stem input [n][w][w][cin_pad] from window
 *   crops (+ renoise, conditioning planes, mask, constant plane) and x_noisy;
 * ig_unet_output: Phi[n][C][h][w] = c_skip * x_noisy + c_out * F[..., c];
 * ig_unet_out_head: the output conv fused with it: F = conv3x3(xa, w_out)
 *   ([cout_pad][9][64] bf16, rows >= C zero) in f32, never stored (cin 64,
 *   C <= 8, w % 128 == 0, h % 4 == 0);
 * ig_avgpool2_bf16: 2x2 mean -> out and mp_silu(out);
 * ig_upsample2_bf16: nearest 2x.
 * layout (pool / upsample): bit 0 input, bit 1 output in the gutter layout
 * [n][h][w+2][c] of ig_conv_params_t.gutter (zero columns written). */
int ig_unet_gather_input(const float* src, int32_t src_batched, int64_t src_x0, int64_t src_y0,
                         int32_t src_w, int32_t src_h, int32_t channels, const int64_t* wxy,
                         int32_t n, const float* cond_parent, int64_t cond_x0, int64_t cond_y0,
                         int32_t cond_w, int32_t cond_h, int32_t cond_c, int32_t cond_scale,
                         int32_t cond_mask_channel, uint64_t cond_seed, uint64_t renoise_seed,
                         uint32_t renoise_stream, float sigma, float c_in, int32_t first_step,
                         void* x_in, int32_t window, int32_t cin_pad, int32_t in_planes,
                         float* x_noisy, void* cuda_stream);
int ig_unet_output(const void* f, int32_t n, int32_t h, int32_t w, int32_t fc,
                   const float* x_noisy, int32_t channels, float c_skip, float c_out,
                   int32_t flags, float* out, void* cuda_stream);
int ig_unet_out_head(const void* xa, int32_t n, int32_t h, int32_t w, int32_t cin,
                     const void* w_out, int32_t cout_pad, int32_t channels, const float* x_noisy,
                     float c_skip, float c_out, float* out, void* cuda_stream);
/* EDM2 self-attention over n windows of hw tokens (NHWC, c channels, heads of
 * 64): ig_attn_prep unit-RMS-normalises q, k (bf16) and v in place per token
 * and head -- q additionally carries the softmax scale 1/8 * log2 e and v is
 * rewritten as f16 -- and writes the normalised v transposed ([n][c/64][64][hw],
 * bf16) when vt != NULL.  (The UNet produces the same operands from the q/k/v
 * conv epilogues, ig_conv_params_t.head_norm.)  ig_attention computes
 * y = softmax(q k^T / 8) v per head (bf16 out): tcgen05, S and O in TMEM, P = 2^s
 * in f16, V read as an MN-major operand, the row sums from a ones block in the
 * PV MMA.  hw % 8 == 0 (partial 128-token tiles masked). */
int ig_attn_prep(void* q, void* k, void* v, int32_t n, int32_t hw, int32_t c, void* vt,
                 void* cuda_stream);
int ig_attention(const void* q, const void* k, const void* v, int32_t n, int32_t hw, int32_t c,
                 void* y, void* cuda_stream);
int ig_avgpool2_bf16(const void* in, int32_t n, int32_t h, int32_t w, int32_t c, void* out,
                     void* out_act, int32_t layout, void* cuda_stream);
int ig_upsample2_bf16(const void* in, int32_t n, int32_t h, int32_t w, int32_t c, void* out,
                      int32_t layout, void* cuda_stream);
/* Fused UNet input gather + stem convolution (64 output channels): builds the
 * tap-packed input planes of each 128-pixel tile in SMEM (window crops of the
 * source canvas/batch, consistency renoise, conditioning + mask, constant
 * plane), runs the stem GEMM on the tensor cores and writes x and mp_silu(x)
 * (bf16 NHWC [n][window][window][64]) plus x_noisy (f32 [n][channels][w][w]).
 * Same input-plane contract as ig_unet_gather_input. */
int ig_unet_stem(const float* src, int32_t src_batched, int64_t src_x0, int64_t src_y0,
                 int32_t src_w, int32_t src_h, int32_t channels, const int64_t* wxy, int32_t n,
                 const float* cond_parent, int64_t cond_x0, int64_t cond_y0, int32_t cond_w,
                 int32_t cond_h, int32_t cond_c, int32_t cond_scale, int32_t cond_mask_channel,
                 uint64_t cond_seed, uint64_t renoise_seed, uint32_t renoise_stream, float sigma,
                 float c_in, int32_t first_step, int32_t window, int32_t in_planes,
                 const void* w_stem, float act_gain, void* out_x, void* out_xa, float* x_noisy,
                 void* cuda_stream);
/* same contract on CUDA cores (fp32 accumulate, identical epilogue); used by
 * the tests as an independent device cross-check of the tensor-core kernel */
int ig_conv_simt(const ig_conv_params_t* p, void* cuda_stream);

#ifdef __cplusplus
}
#endif
#endif /* INFIGRID_B200_H */
