// infigrid_b200 core kernels: noise (K1), analytic Phi (K3), canonical blend
// (K5), elevation transforms (K6), features / conditioning / base maps (K7-K9).
//
// Every kernel here is on the bit-exact parity path: arithmetic goes through
// explicitly rounded intrinsics (ig::radd/rmul/...) in the order the
// reference's numpy expressions evaluate, and the file is compiled with
// -fmad=false as a second guard.  Reference citations are per kernel.
#include <cstdarg>
#include <atomic>
#include <cstring>

#include <cuda.h>
#include <cuda_fp16.h>
#include <type_traits>

#include "ig_common.cuh"
#include "ig_noise.cuh"

namespace ig {

static thread_local char g_err[512] = {0};

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

static std::atomic<long long> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

static inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// =====================================================================
// K1 noise_region  (noise.py:74-86)
// Each thread produces 4 consecutive x samples of one row; the 4 outputs
// are stored together (16 B for f32) when the row is 4-aligned.
template <typename T>
__global__ void __launch_bounds__(256) noise_region_kernel(uint64_t prefix, int64_t x0, int64_t y0,
                                                           int32_t w, int32_t h, int32_t ch0,
                                                           int32_t nch, T* __restrict__ out,
                                                           int32_t* slow_count) {
  const int64_t quads_per_row = (w + 3) / 4;
  const int64_t total = quads_per_row * h * nch;
  int slow = 0;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = q / quads_per_row;      // c*h + py
    const int32_t px0 = (int32_t)(q - row * quads_per_row) * 4;
    const int32_t c = (int32_t)(row / h);
    const int32_t py = (int32_t)(row - (int64_t)c * h);
    const int64_t Y = y0 + py;
    float v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      v[k] = 0.f;
      if (px0 + k < w) v[k] = noise_value(prefix, x0 + px0 + k, Y, (uint32_t)(ch0 + c), &slow);
    }
    T* dst = out + row * w + px0;
    if (sizeof(T) == 4 && (w & 3) == 0) {
      *reinterpret_cast<float4*>(dst) = make_float4(v[0], v[1], v[2], v[3]);
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (px0 + k < w) dst[k] = (T)v[k];
    }
  }
  if (slow_count && __syncthreads_or(slow) && threadIdx.x == 0) atomicAdd(slow_count, 1);
}

// =====================================================================
// K3 analytic Phi  (denoise.py:75-113; box_mean transforms.py:29-51)
struct SrcView {
  const void* base;
  int batched;
  int64_t x0, y0;
  int32_t w, h, channels;
};
struct CondView {
  const void* parent;
  int64_t x0, y0;
  int32_t w, h, c, scale, mask_channel, fill;
  uint64_t prefix;  // noise prefix of (seed, STREAM_CONDITIONING)
};

// value of window k, channel c at window-local (yy, xx) (already clamped)
template <typename T>
__device__ __forceinline__ T src_at(const SrcView& s, const int64_t* wxy, int k, int c, int win,
                                    int yy, int xx) {
  const T* b = reinterpret_cast<const T*>(s.base);
  if (s.batched) return b[(((int64_t)k * s.channels + c) * win + yy) * win + xx];
  const int64_t gx = wxy[2 * k] + xx - s.x0;
  const int64_t gy = wxy[2 * k + 1] + yy - s.y0;
  return b[((int64_t)c * s.h + gy) * s.w + gx];
}

template <typename T>
__global__ void __launch_bounds__(256) phi_analytic_kernel(int kind, int radius, T a_coef, T b_coef,
                                                           int lam_zero, SrcView src,
                                                           const int64_t* __restrict__ wxy, int n,
                                                           int win, CondView cond,
                                                           T* __restrict__ out) {
  const int64_t per_win = (int64_t)src.channels * win * win;
  const int64_t total = per_win * n;
  const T kdiv = (T)(2 * radius + 1);
  int slow = 0;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(idx / per_win);
    int64_t rem = idx - (int64_t)k * per_win;
    const int c = (int)(rem / (win * win));
    rem -= (int64_t)c * win * win;
    const int y = (int)(rem / win), x = (int)(rem - (int64_t)y * win);
    const T xv = src_at<T>(src, wxy, k, c, win, y, x);
    T res;
    if (kind == IG_PHI_IDENTITY || lam_zero) {
      res = xv;
    } else {
      T blur = xv;
      if (radius > 0) {
        // rows (axis -2) first, then columns; clamp-to-edge inside the window
        T hacc = (T)0;
        for (int dx = -radius; dx <= radius; ++dx) {
          int xx = min(max(x + dx, 0), win - 1);
          T vacc = (T)0;
          for (int dy = -radius; dy <= radius; ++dy) {
            int yy = min(max(y + dy, 0), win - 1);
            vacc = radd(vacc, src_at<T>(src, wxy, k, c, win, yy, xx));
          }
          hacc = radd(hacc, rdiv(vacc, kdiv));
        }
        blur = rdiv(hacc, kdiv);
      }
      res = radd(rmul(a_coef, xv), rmul(b_coef, blur));
    }
    if (kind == IG_PHI_COND_AFFINE && cond.parent != nullptr) {
      // conditioning_for_window (denoise.py:116-163): NN upsample of the
      // coarse parent's channel 0; holes (mask < 1) take stream-101 noise
      const int64_t X = wxy[2 * k] + x, Y = wxy[2 * k + 1] + y;
      const int64_t cx = floordiv(X, cond.scale) - cond.x0;
      const int64_t cy = floordiv(Y, cond.scale) - cond.y0;
      const T* par = reinterpret_cast<const T*>(cond.parent);
      const int64_t plane = (int64_t)cond.w * cond.h;
      T m = (T)1;
      if (cond.mask_channel >= 0) m = par[cond.mask_channel * plane + cy * cond.w + cx];
      T target = par[cy * cond.w + cx];
      if (cond.fill && m < (T)1) target = (T)noise_value(cond.prefix, X, Y, 0u, &slow);
      res = radd(res, rmul(m, rsub(target, res)));
    }
    out[idx] = res;
  }
}

// Tiled form of phi_analytic_kernel: one CTA = one band of `band` rows of one
// (window, channel) plane, full window width.  The clamped source rows
// (band + 2r) are staged in SMEM once; the blur is evaluated separably with the
// reference's own rounding sequence (transforms.py:29-51 sums axis -2 first,
// and each column sum is divided by k before the horizontal sum), so
//   D[y][x'] = rdiv(sum_dy S[y+dy][x'], k)     (once per pixel, not per tap)
//   blur     = rdiv(sum_dx D[y][clamp(x+dx)], k)
// is the same operation sequence per output as the direct form above:
// bit-identical, with 2(2r+1) adds + 2 divisions per pixel instead of
// (2r+1)^2 + 2r+2 and 32-bit indexing throughout.
// Threads own fixed columns (TX = min(win, 256) lanes across, TY row groups)
// and walk rows, so the clamped neighbour columns are computed once per
// column, not per pixel.  R >= 0: the effective radius as a template constant
// (the sampler's radius 0 / 1 cases); R = -1: runtime radius.
template <typename T, int R>
__global__ void __launch_bounds__(256) phi_tile_kernel(int kind, int radius, T a_coef, T b_coef,
                                                       int lam_zero, SrcView src,
                                                       const int64_t* __restrict__ wxy, int win,
                                                       int band, CondView cond,
                                                       T* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char phi_smem[];
  const bool plain = kind == IG_PHI_IDENTITY || lam_zero;
  const int r = R >= 0 ? R : (plain ? 0 : radius);     // host passes R = effective radius
  const int C = src.channels;
  const int k = blockIdx.y / C, c = blockIdx.y - k * C;
  const int y0 = blockIdx.x * band;
  const int rows = min(band, win - y0);
  const int srows = rows + 2 * r;
  T* S = reinterpret_cast<T*>(phi_smem);                  // (band + 2r) x win, clamped rows
  T* D = S + (size_t)(band + 2 * r) * win;                // band x win column sums / k
  const T kdiv = (T)(2 * r + 1);
  const int TX = win < 256 ? win : 256, TY = 256 / TX;
  const int tx = threadIdx.x % TX, ty = threadIdx.x / TX;
  const bool active = ty < TY;
  const T* base;
  int64_t rs;
  if (src.batched) {
    base = reinterpret_cast<const T*>(src.base) + ((int64_t)k * C + c) * win * win;
    rs = win;
  } else {
    base = reinterpret_cast<const T*>(src.base) +
           ((int64_t)c * src.h + (wxy[2 * k + 1] - src.y0)) * src.w + (wxy[2 * k] - src.x0);
    rs = src.w;
  }
  if (active) {
    // 8 independent loads in flight per thread before the SMEM stores
    for (int x = tx; x < win; x += TX)
      for (int i0 = ty; i0 < srows; i0 += 8 * TY) {
        T v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int i = i0 + u * TY;
          if (i < srows) v[u] = base[(int64_t)min(max(y0 - r + i, 0), win - 1) * rs + x];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (i0 + u * TY < srows) S[(i0 + u * TY) * win + x] = v[u];
      }
  }
  __syncthreads();
  if (r > 0) {
    if (active)
      for (int x = tx; x < win; x += TX)
        for (int yl = ty; yl < rows; yl += TY) {
          T vacc = (T)0;
          for (int dy = 0; dy <= 2 * r; ++dy) vacc = radd(vacc, S[(yl + dy) * win + x]);
          D[yl * win + x] = rdiv(vacc, kdiv);
        }
    __syncthreads();
  }
  if (!active) return;
  int slow = 0;
  T* obase = out + (((int64_t)k * C + c) * win + y0) * win;
  for (int x = tx; x < win; x += TX) {
    int xm[R > 0 ? 2 * R + 1 : 1];
    if (R > 0) {
#pragma unroll
      for (int d = 0; d < (R > 0 ? 2 * R + 1 : 1); ++d) xm[d] = min(max(x + d - R, 0), win - 1);
    }
    for (int yl = ty; yl < rows; yl += TY) {
      const T xv = S[(yl + r) * win + x];
      T res;
      if (plain) {
        res = xv;
      } else {
        T blur = xv;
        if (r > 0) {
          T hacc = (T)0;
          if (R > 0) {
#pragma unroll
            for (int d = 0; d < (R > 0 ? 2 * R + 1 : 1); ++d) hacc = radd(hacc, D[yl * win + xm[d]]);
          } else {
            for (int dx = -r; dx <= r; ++dx)
              hacc = radd(hacc, D[yl * win + min(max(x + dx, 0), win - 1)]);
          }
          blur = rdiv(hacc, kdiv);
        }
        res = radd(rmul(a_coef, xv), rmul(b_coef, blur));
      }
      if (kind == IG_PHI_COND_AFFINE && cond.parent != nullptr) {
        const int64_t X = wxy[2 * k] + x, Y = wxy[2 * k + 1] + y0 + yl;
        const int64_t cx = floordiv(X, cond.scale) - cond.x0;
        const int64_t cy = floordiv(Y, cond.scale) - cond.y0;
        const T* par = reinterpret_cast<const T*>(cond.parent);
        const int64_t plane = (int64_t)cond.w * cond.h;
        T m = (T)1;
        if (cond.mask_channel >= 0) m = par[cond.mask_channel * plane + cy * cond.w + cx];
        T target = par[cy * cond.w + cx];
        if (cond.fill && m < (T)1) target = (T)noise_value(cond.prefix, X, Y, 0u, &slow);
        res = radd(res, rmul(m, rsub(target, res)));
      }
      obase[yl * win + x] = res;
    }
  }
}

// =====================================================================
// K5 blend  (store.py:428-436 _accumulate, sampler.py:151-154, store.py:549-554)
// Gather form: each output pixel walks its covering windows in canonical
// (j, i) order and sums their contributions starting from +0, exactly the
// per-pixel sequence of the reference's scatter-add loop.  No atomics.
template <typename T>
__global__ void __launch_bounds__(256) blend_kernel(const T* const* __restrict__ win_data,
                                                    int64_t i0, int64_t j0, int ni, int nj,
                                                    int win, int stride, int64_t ox, int64_t oy,
                                                    int channels, int mode,
                                                    const T* __restrict__ weight, int64_t rx0,
                                                    int64_t ry0, int rw, int rh, int divide,
                                                    T* __restrict__ out) {
  // one output row per blockIdx.y, 256 columns per thread-row pass: the window
  // rows covering the row (j range, local y) are per-block constants and the
  // per-pixel window columns come from 32-bit quotient/remainder arithmetic
  // (no 64-bit division per pixel).  Same per-pixel accumulation order as the
  // reference's scatter-add: windows in canonical (j asc, i asc) order from +0.
  const int64_t npix = (int64_t)rw * rh;
  for (int py = blockIdx.y; py < rh; py += gridDim.y) {
  const int64_t Y = ry0 + py;
  int64_t jlo = ceildiv(Y - oy - win + 1, stride), jhi = floordiv(Y - oy, stride);
  jlo = jlo > j0 ? jlo : j0;
  jhi = jhi < j0 + nj - 1 ? jhi : j0 + nj - 1;
  const int nrows = jhi >= jlo ? (int)(jhi - jlo + 1) : 0;
  // column origin of this block's first pixel relative to the layout
  const int px_begin = blockIdx.x * 1024;
  const int64_t X0 = rx0 + px_begin;
  const int64_t base = floordiv(X0 - ox, stride);             // window column index of X0
  const int r0 = (int)((X0 - ox) - base * stride);           // 0 .. stride-1
  const int out_planes = mode == 1 ? channels + 1 : channels;
  for (int px = px_begin + threadIdx.x; px < rw && px < px_begin + 1024; px += blockDim.x) {
    const int t = r0 + (px - px_begin);
    const int q = t / stride, rr = t - q * stride;            // X - ox = (base + q) * stride + rr
    // covering windows i = base + q - m with lx = rr + m * stride < win, m >= 0
    int mmax = (win - 1 - rr) / stride;                       // largest m with lx < win
    const int64_t ihi_raw = base + q;
    int64_t ilo = ihi_raw - mmax, ihi = ihi_raw;
    if (ilo < i0) ilo = i0;
    if (ihi > i0 + ni - 1) ihi = i0 + ni - 1;
    const int64_t p = (int64_t)py * rw + px;
    // window columns relative to the table: ii = i - i0 in [iilo, iihi]
    const int iilo = (int)(ilo - i0), iihi = (int)(ihi - i0), ihr = (int)(ihi_raw - i0);
    if (mode == 1 && channels <= 4) {
      // one pass: the weight sum and every channel's weighted sum, each in the
      // canonical (j asc, i asc) order (the chains are independent)
      T wsum = (T)0, acc[4] = {(T)0, (T)0, (T)0, (T)0};
      for (int jj = 0; jj < nrows; ++jj) {
        const int64_t j = jlo + jj;
        const int ly = (int)(Y - (j * stride + oy));
        const T* wrow = weight + (int64_t)ly * win;
        const T* const* dptr = win_data + (j - j0) * ni;
        for (int ii = iilo; ii <= iihi; ++ii) {
          const T* d = dptr[ii];
          if (!d) continue;
          const int lx = rr + (ihr - ii) * stride;
          const T wv = wrow[lx];
          wsum = radd(wsum, wv);
          const T* dp = d + (int64_t)ly * win + lx;
#pragma unroll
          for (int c = 0; c < 4; ++c)
            if (c < channels) acc[c] = radd(acc[c], rmul(wv, dp[(int64_t)c * win * win]));
        }
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (c >= channels) break;
        if (divide)
          out[(int64_t)c * npix + p] = wsum > (T)0 ? rdiv(acc[c], wsum) : (T)0;
        else
          out[(int64_t)c * npix + p] = acc[c];
      }
      if (!divide) out[(int64_t)channels * npix + p] = wsum;
    } else if (mode == 1) {
      T wsum = (T)0;
      for (int jj = 0; jj < nrows; ++jj) {
        const int64_t j = jlo + jj;
        const int ly = (int)(Y - (j * stride + oy));
        const T* wrow = weight + (int64_t)ly * win;
        const T* const* dptr = win_data + (j - j0) * ni;
        for (int64_t i = ilo; i <= ihi; ++i) {
          if (!dptr[i - i0]) continue;
          const int lx = rr + (int)(ihi_raw - i) * stride;
          wsum = radd(wsum, wrow[lx]);
        }
      }
      for (int c = 0; c < channels; ++c) {
        T acc = (T)0;
        for (int jj = 0; jj < nrows; ++jj) {
          const int64_t j = jlo + jj;
          const int ly = (int)(Y - (j * stride + oy));
          const T* wrow = weight + (int64_t)ly * win;
          const T* const* dptr = win_data + (j - j0) * ni;
          for (int64_t i = ilo; i <= ihi; ++i) {
            const T* d = dptr[i - i0];
            if (!d) continue;
            const int lx = rr + (int)(ihi_raw - i) * stride;
            acc = radd(acc, rmul(wrow[lx], d[((int64_t)c * win + ly) * win + lx]));
          }
        }
        if (divide)
          out[(int64_t)c * npix + p] = wsum > (T)0 ? rdiv(acc, wsum) : (T)0;
        else
          out[(int64_t)c * npix + p] = acc;
      }
      if (!divide) out[(int64_t)channels * npix + p] = wsum;
    } else {
      for (int c = 0; c < out_planes; ++c) {
        T acc = (T)0;
        for (int jj = 0; jj < nrows; ++jj) {
          const int64_t j = jlo + jj;
          const int ly = (int)(Y - (j * stride + oy));
          const T* const* dptr = win_data + (j - j0) * ni;
          for (int64_t i = ilo; i <= ihi; ++i) {
            const T* d = dptr[i - i0];
            if (!d) continue;
            const int lx = rr + (int)(ihi_raw - i) * stride;
            acc = radd(acc, d[((int64_t)c * win + ly) * win + lx]);
          }
        }
        out[(int64_t)c * npix + p] = acc;
      }
    }
  }
  }   // rows
}

// Fast path for window == 2 * stride (every sampler layout): the pixels of
// one stride x stride CELL of the layout lattice are covered by the same four
// windows, (cj-1, ci-1), (cj-1, ci), (cj, ci-1), (cj, ci) in canonical order,
// at fixed local offsets.  One CTA = P passes of (256 / (stride/4)) rows of one
// cell; a thread handles 4 consecutive pixels per pass with 16-byte loads.
// Every load of every pass is issued before the first add (absent windows and
// out-of-region passes load a valid dummy address and are masked afterwards),
// so a warp keeps P * 4 * (1 + C) 16-byte requests in flight -- the kernel is
// latency-bound otherwise (ncu: long-scoreboard stalls, 2.6 TB/s).  Same
// per-pixel sums in the same order as blend_kernel (absent windows skipped).
template <typename T>
__device__ __forceinline__ void ld4(const T* p, T (&v)[4]) {
  if (sizeof(T) == 4) {
    const float4 f = __ldg(reinterpret_cast<const float4*>(p));
    v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
  } else {
    const double2 a = __ldg(reinterpret_cast<const double2*>(p));
    const double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
  }
}

template <typename T, int C>
constexpr int blend_cells_passes() { return sizeof(T) * C <= 8 ? 2 : 1; }

template <typename T, int C>
__global__ void __launch_bounds__(256) blend_cells_kernel(
    const T* const* __restrict__ win_data, int64_t i0, int64_t j0, int ni, int nj, int win,
    int stride, int64_t ox, int64_t oy, const T* __restrict__ weight, int64_t rx0,
    int64_t ry0, int rw, int rh, int divide, int64_t ci_lo, int64_t cj_lo, int ncx,
    T* __restrict__ out) {
  constexpr int P = blend_cells_passes<T, C>();
  __shared__ const T* s_wp[4];
  const int64_t npix = (int64_t)rw * rh;
  const int q4 = stride / 4;                          // quads per cell row
  const int rows_per_pass = 256 / q4;                 // cell rows per pass of the CTA
  const int rows_per_cta = P * rows_per_pass;
  const int blocks_per_cell = stride / rows_per_cta;
  const int cell = blockIdx.x / blocks_per_cell;
  const int rb = blockIdx.x - cell * blocks_per_cell;
  const int64_t ci = ci_lo + cell % ncx, cj = cj_lo + cell / ncx;
  if (threadIdx.x < 4) {        // the 4 candidate windows (canonical order), once per CTA
    const int64_t j = cj - 1 + (threadIdx.x >> 1), i = ci - 1 + (threadIdx.x & 1);
    const bool in = j >= j0 && j < j0 + nj && i >= i0 && i < i0 + ni;
    s_wp[threadIdx.x] = in ? win_data[(j - j0) * ni + (i - i0)] : nullptr;
  }
  __syncthreads();
  const T* wp[4] = {s_wp[0], s_wp[1], s_wp[2], s_wp[3]};
  const int v = (threadIdx.x % q4) * 4;                        // first column of the quad
  const int plane = win * win;
  T wv[P][4][4], dv[P][4][C][4];
  int py[P], px[P];
  bool ok[P];
#pragma unroll
  for (int pass = 0; pass < P; ++pass) {
    const int u = rb * rows_per_cta + pass * rows_per_pass + threadIdx.x / q4;   // cell row
    py[pass] = (int)(cj * stride + oy + u - ry0);
    px[pass] = (int)(ci * stride + ox + v - rx0);
    ok[pass] = !(py[pass] < 0 || py[pass] >= rh || px[pass] + 3 < 0 || px[pass] >= rw);
#pragma unroll
    for (int w4 = 0; w4 < 4; ++w4) {
      const int lofs = (u + (1 - (w4 >> 1)) * stride) * win + v + (1 - (w4 & 1)) * stride;
      ld4(weight + lofs, wv[pass][w4]);
      const bool use = ok[pass] && wp[w4] != nullptr;
#pragma unroll
      for (int c = 0; c < C; ++c)
        ld4(use ? wp[w4] + (int64_t)c * plane + lofs : weight + lofs, dv[pass][w4][c]);
    }
  }
#pragma unroll
  for (int pass = 0; pass < P; ++pass) {
    if (!ok[pass]) continue;
    T wsum[4] = {(T)0, (T)0, (T)0, (T)0};
    T acc[C][4];
#pragma unroll
    for (int c = 0; c < C; ++c)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[c][e] = (T)0;
#pragma unroll
    for (int w4 = 0; w4 < 4; ++w4) {
      if (!wp[w4]) continue;
#pragma unroll
      for (int e = 0; e < 4; ++e) wsum[e] = radd(wsum[e], wv[pass][w4][e]);
#pragma unroll
      for (int c = 0; c < C; ++c)
#pragma unroll
        for (int e = 0; e < 4; ++e)
          acc[c][e] = radd(acc[c][e], rmul(wv[pass][w4][e], dv[pass][w4][c][e]));
    }
    const bool full = px[pass] >= 0 && px[pass] + 3 < rw;
    const int64_t p = (int64_t)py[pass] * rw + px[pass];
#pragma unroll
    for (int c = 0; c <= C; ++c) {
      if (c == C && divide) break;
      T o[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (c == C) o[e] = wsum[e];
        else if (divide) o[e] = wsum[e] > (T)0 ? rdiv(acc[c < C ? c : 0][e], wsum[e]) : (T)0;
        else o[e] = acc[c < C ? c : 0][e];
      }
      T* dst = out + (int64_t)c * npix + p;
      if (full && sizeof(T) == 4 && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
        *reinterpret_cast<float4*>(dst) = make_float4((float)o[0], (float)o[1], (float)o[2],
                                                      (float)o[3]);
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (px[pass] + e >= 0 && px[pass] + e < rw) dst[e] = o[e];
      }
    }
  }
}

template <typename T, int C>
static void launch_blend_cells(const void* const* win_data, int64_t i0, int64_t j0, int ni,
                               int nj, int window, int stride, int64_t ox, int64_t oy,
                               const void* weight, int64_t rx0, int64_t ry0, int rw, int rh,
                               int divide, int64_t ci_lo, int64_t cj_lo, int ncx, int64_t cells,
                               void* out, cudaStream_t st) {
  const int rows_per_cta = blend_cells_passes<T, C>() * (256 / (stride / 4));
  const int64_t ctas = cells * (stride / rows_per_cta);
  blend_cells_kernel<T, C><<<(unsigned)ctas, 256, 0, st>>>(
      (const T* const*)win_data, i0, j0, ni, nj, window, stride, ox, oy, (const T*)weight, rx0,
      ry0, rw, rh, divide, ci_lo, cj_lo, ncx, (T*)out);
  note_launch();
}

template <typename T>
__global__ void divide_weighted_kernel(const T* __restrict__ raw, int channels, int64_t npix,
                                       T* __restrict__ out) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < npix;
       p += (int64_t)gridDim.x * blockDim.x) {
    const T w = raw[(int64_t)channels * npix + p];
    for (int c = 0; c < channels; ++c)
      out[(int64_t)c * npix + p] = w > (T)0 ? rdiv(raw[(int64_t)c * npix + p], w) : (T)0;
  }
}

// =====================================================================
// K6 transforms  (transforms.py:17-114)
template <typename T>
__global__ void box_mean_kernel(const T* __restrict__ in, int planes, int h, int w, int radius,
                                T* __restrict__ out) {
  const int64_t total = (int64_t)planes * h * w;
  const T kdiv = (T)(2 * radius + 1);
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pl = idx / ((int64_t)h * w);
    const int rem = (int)(idx - pl * h * w);
    const int y = rem / w, x = rem - y * w;
    const T* P = in + pl * h * w;
    if (radius == 0) { out[idx] = P[rem]; continue; }
    T hacc = (T)0;
    for (int dx = -radius; dx <= radius; ++dx) {
      const int xx = min(max(x + dx, 0), w - 1);
      T vacc = (T)0;
      for (int dy = -radius; dy <= radius; ++dy) {
        const int yy = min(max(y + dy, 0), h - 1);
        vacc = radd(vacc, P[yy * w + xx]);
      }
      hacc = radd(hacc, rdiv(vacc, kdiv));
    }
    out[idx] = rdiv(hacc, kdiv);
  }
}

template <typename TI>
__global__ void widen_kernel(const TI* __restrict__ in, int64_t n, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (double)in[i];
}

// numpy pairwise summation (numpy/_core/src/umath/loops_utils.h.src) of
// v(s..s+n): blocks of <8 sequentially from -0.0, <=128 with 8 running
// partial sums folded as a tree, larger blocks split at an 8-aligned half.
template <typename T, typename F>
__device__ T np_pairwise(const F& v, int s, int n) {
  if (n < 8) {
    T res = (T)-0.0;
    for (int i = 0; i < n; ++i) res = radd(res, v(s + i));
    return res;
  }
  if (n <= 128) {
    T r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = v(s + j);
    int i = 8;
    for (; i < n - (n % 8); i += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = radd(r[j], v(s + i + j));
    }
    T res = radd(radd(radd(r[0], r[1]), radd(r[2], r[3])), radd(radd(r[4], r[5]), radd(r[6], r[7])));
    for (; i < n; ++i) res = radd(res, v(s + i));
    return res;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  return radd(np_pairwise<T>(v, s, n2), np_pairwise<T>(v, s + n2, n - n2));
}

// block_mean of blur3_iterated input (transforms.py:54-67), float64.
// numpy order for .mean(axis=(-3,-1)) of the (h/f, f, w/f, f) view: for each
// of the f block rows (outer, sequential, starting from 0) add the pairwise
// sum of that row's f values; then divide by f*f.
template <typename T>
__global__ void block_mean_kernel(const T* __restrict__ in, int planes, int h, int w, int f,
                                  T* __restrict__ low) {
  const int lh = h / f, lw = w / f;
  const int64_t total = (int64_t)planes * lh * lw;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pl = idx / ((int64_t)lh * lw);
    const int rem = (int)(idx - pl * lh * lw);
    const int by = rem / lw, bx = rem - by * lw;
    const T* P = in + pl * h * w + (int64_t)(by * f) * w + bx * f;
    T s = (T)0;
    for (int r = 0; r < f; ++r) {
      const T* row = P + (int64_t)r * w;
      s = radd(s, np_pairwise<T>([&](int i) { return row[i]; }, 0, f));
    }
    low[idx] = rdiv(s, (T)(f * f));
  }
}

template <typename TI>
__global__ void __launch_bounds__(256, 4) blur_block_mean_tile_kernel(
    const TI* __restrict__ in, int h, int w, int r, int f, int TH, int TW,
    double* __restrict__ low) {
  extern __shared__ __align__(16) unsigned char bbm_smem[];
  double* S = reinterpret_cast<double*>(bbm_smem);             // (TH+2r) x (TW+2r)
  double* D = S + (size_t)(TH + 2 * r) * (TW + 2 * r);        // TH x (TW+2r); then row sums
  const int pl = blockIdx.z;
  const int ty0 = blockIdx.y * TH, tx0 = blockIdx.x * TW;
  const int rows = min(TH, h - ty0), cols = min(TW, w - tx0);
  const int SW = cols + 2 * r, SH = rows + 2 * r;
  const TI* P = in + (int64_t)pl * h * w;
  {
    const int total = SH * SW;
    for (int e0 = threadIdx.x; e0 < total; e0 += 8 * 256) {
      TI v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * 256;
        if (e < total) {
          const int i = e / SW, j = e - i * SW;
          const int gy = min(max(ty0 - r + i, 0), h - 1), gx = min(max(tx0 - r + j, 0), w - 1);
          v[u] = P[(int64_t)gy * w + gx];
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (e0 + u * 256 < total) S[e0 + u * 256] = (double)v[u];
    }
  }
  __syncthreads();
  // B: rows x cols; after a blur it is stored with one pad double per f-wide
  // segment (seg stride f+1) so the row-sum lanes below hit distinct banks
  double* B = S;
  const bool pad = r > 0 && (size_t)rows * (cols + cols / f) <= (size_t)SH * SW;
  const int segw = pad ? f + 1 : f, ldb = (cols / f) * segw;
  if (r > 0) {
    const double k = (double)(2 * r + 1);
    for (int e = threadIdx.x; e < rows * SW; e += 256) {
      const int i = e / SW, j = e - i * SW;
      double vacc = 0.0;
      for (int dy = 0; dy <= 2 * r; ++dy) vacc = radd(vacc, S[(i + dy) * SW + j]);
      D[e] = rdiv(vacc, k);
    }
    __syncthreads();
    // B overwrites S: S is dead once D exists (the barrier above)
    for (int e = threadIdx.x; e < rows * cols; e += 256) {
      const int i = e / cols, j = e - i * cols;
      double hacc = 0.0;
      for (int dx = 0; dx <= 2 * r; ++dx) hacc = radd(hacc, D[i * SW + j + dx]);
      const int seg = j / f;
      B[i * ldb + seg * segw + (j - seg * f)] = rdiv(hacc, k);
    }
    __syncthreads();
  }
  // row sums of every (block, block row) -> D, then the block means
  // (block fastest across lanes: row sum t = rr * nblk + blk)
  const int nbx = cols / f, nby = rows / f, nblk = nbx * nby;
  for (int t = threadIdx.x; t < nblk * f; t += 256) {
    const int rr = t / nblk, blk = t - rr * nblk;
    const int by = blk / nbx, bx = blk - by * nbx;
    const double* row = B + (by * f + rr) * ldb + bx * segw;
    D[t] = np_pairwise<double>([&](int i) { return row[i]; }, 0, f);
  }
  __syncthreads();
  const int lw = w / f;
  for (int blk = threadIdx.x; blk < nblk; blk += 256) {
    const int by = blk / nbx, bx = blk - by * nbx;
    double s = 0.0;
    for (int rr = 0; rr < f; ++rr) s = radd(s, D[rr * nblk + blk]);
    low[((int64_t)pl * (h / f) + ty0 / f + by) * lw + tx0 / f + bx] = rdiv(s, (double)(f * f));
  }
}

// Residual / merge on a 2-D grid: blockIdx.y = plane row, 4 pixels per thread
// with a stride of 256 (coalesced), 32-bit indexing, shift for power-of-two f.
template <typename TX>
__global__ void __launch_bounds__(256) laplacian_residual_rows_kernel(
    const TX* __restrict__ x, const double* __restrict__ low, int planes, int h, int w, int f,
    double* __restrict__ high) {
  const int lw = w / f;
  const int sh = (f & (f - 1)) == 0 ? __ffs(f) - 1 : -1;
  for (int64_t prow = blockIdx.y; prow < (int64_t)planes * h; prow += gridDim.y) {
    const int pl = (int)(prow / h), y = (int)(prow - (int64_t)pl * h);
    const double* lrow = low + ((int64_t)pl * (h / f) + (sh >= 0 ? y >> sh : y / f)) * lw;
    const int64_t base = prow * w;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int xx = blockIdx.x * 1024 + e * 256 + threadIdx.x;
      if (xx < w)
        high[base + xx] = rsub((double)x[base + xx], lrow[sh >= 0 ? xx >> sh : xx / f]);
    }
  }
}

// element conversions: exact widenings (f16/f32/ints -> f64, f16 -> f32) and the
// round-to-nearest narrowings numpy's astype performs (f32 -> f16, f64 -> f32);
// float -> int truncates toward zero like numpy's C cast
template <typename TO, typename TI>
__device__ __forceinline__ TO convert_elem(TI v) {
  if constexpr (std::is_same<TI, __half>::value) {
    return convert_elem<TO>(__half2float(v));
  } else if constexpr (std::is_same<TO, __half>::value) {
    if constexpr (std::is_same<TI, double>::value) return __double2half(v);
    else return __float2half_rn((float)v);
  } else {
    return (TO)v;
  }
}

template <typename TO, typename TI>
__global__ void convert_kernel(const TI* __restrict__ in, int64_t n, TO* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = convert_elem<TO>(in[i]);
}

template <typename TO>
__global__ void __launch_bounds__(256) laplacian_merge_rows_kernel(
    const double* __restrict__ low, const double* __restrict__ high, int planes, int h, int w,
    int f, int square_out, TO* __restrict__ out) {
  const int lw = w / f;
  const int sh = (f & (f - 1)) == 0 ? __ffs(f) - 1 : -1;
  for (int64_t prow = blockIdx.y; prow < (int64_t)planes * h; prow += gridDim.y) {
    const int pl = (int)(prow / h), y = (int)(prow - (int64_t)pl * h);
    const double* lrow = low + ((int64_t)pl * (h / f) + (sh >= 0 ? y >> sh : y / f)) * lw;
    const int64_t base = prow * w;
    double hv[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int xx = blockIdx.x * 1024 + e * 256 + threadIdx.x;
      hv[e] = xx < w ? high[base + xx] : 0.0;
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int xx = blockIdx.x * 1024 + e * 256 + threadIdx.x;
      if (xx >= w) continue;
      const double sum = radd(lrow[sh >= 0 ? xx >> sh : xx / f], hv[e]);
      if constexpr (std::is_floating_point<TO>::value) {
        TO v = (TO)sum;
        if (square_out) {
          const TO sg = v > (TO)0 ? (TO)1 : (v < (TO)0 ? (TO)-1 : (v == (TO)0 ? (TO)0 : v));
          v = rmul(rmul(sg, v), v);
        }
        out[base + xx] = v;
      } else {
        out[base + xx] = convert_elem<TO>(sum);   // astype(original dtype)
      }
    }
  }
}

// nearest-neighbour replication on the last two axes (transforms.py:70-72),
// element-size generic: one thread per output element of a row segment
template <typename E>
__global__ void upsample_nn_kernel(const E* __restrict__ in, int64_t planes, int h, int w, int f,
                                   E* __restrict__ out) {
  const int64_t W = (int64_t)w * f;
  const int64_t total = planes * h * f * W;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / W;                 // plane * (h*f) + Y
    const int64_t X = i - row * W;
    const int64_t pl = row / ((int64_t)h * f);
    const int64_t Y = row - pl * h * f;
    out[i] = in[(pl * h + Y / f) * w + X / f];
  }
}

template <typename T>
__global__ void signed_square_int_kernel(const T* __restrict__ in, int64_t n, T* __restrict__ out) {
  // np.sign(x) * x * x in the integer dtype (two's-complement wraparound)
  using U = typename std::make_unsigned<T>::type;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const T v = in[i];
    const T sg = v > 0 ? (T)1 : (v < 0 ? (T)-1 : (T)0);
    out[i] = (T)((U)((U)sg * (U)v) * (U)v);
  }
}

template <typename T>
__global__ void signed_pow_kernel(const T* __restrict__ in, int64_t n, int op, T* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const T v = in[i];
    const T sg = v > (T)0 ? (T)1 : (v < (T)0 ? (T)-1 : (v == (T)0 ? (T)0 : v));  // np.sign: +0, nan
    if (op == 0) out[i] = rmul(sg, sqrt(fabs(v)));
    else out[i] = rmul(rmul(sg, v), v);
  }
}

// =====================================================================
// K7 coarse_patch_features  (denoise.py:166-185)
template <typename T>
__global__ void patch_features_kernel(const T* __restrict__ in, int64_t tile_stride, int n,
                                      int h, int w, int p, int rank, T* __restrict__ out) {
  const int oh = h / p, ow = w / p;
  const int64_t total = (int64_t)n * oh * ow;
  const int np2 = p * p;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(idx / ((int64_t)oh * ow));
    const int rem = (int)(idx - (int64_t)k * oh * ow);
    const int by = rem / ow, bx = rem - by * ow;
    const T* P = in + (int64_t)k * tile_stride + (int64_t)(by * p) * w + bx * p;
    auto val = [&](int q) { return P[(q / p) * w + (q % p)]; };
    const T sum = radd((T)0, np_pairwise<T>(val, 0, np2));  // reduce starts at +0
    const T mean = rdiv(sum, (T)np2);
    // rank-th smallest (1-based) with stable tie order == np.sort()[rank-1]
    T sel = val(0);
    for (int q = 0; q < np2; ++q) {
      const T vq = val(q);
      int below = 0, tie_before = 0;
      for (int r = 0; r < np2; ++r) {
        const T vr = val(r);
        below += vr < vq;
        tie_before += (vr == vq) && (r < q);
      }
      if (below + tie_before == rank - 1) { sel = vq; break; }
    }
    T* o = out + (int64_t)k * 3 * oh * ow;
    o[rem] = mean;
    o[(int64_t)oh * ow + rem] = sel;
    o[(int64_t)2 * oh * ow + rem] = (T)1;
  }
}

// =====================================================================
// K8 conditioning_for_window, batched (denoise.py:116-163)
template <typename T>
__global__ void condition_window_kernel(const T* __restrict__ parent, int64_t px0, int64_t py0,
                                        int pw, int ph, int pc, int scale, int mask_channel,
                                        uint64_t prefix, const int64_t* __restrict__ wxy, int n,
                                        int win, T* __restrict__ out, T* __restrict__ mask_out) {
  const int64_t per = (int64_t)win * win;
  const int64_t total = per * n;
  const int64_t plane = (int64_t)pw * ph;
  int slow = 0;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(idx / per);
    const int rem = (int)(idx - (int64_t)k * per);
    const int y = rem / win, x = rem - y * win;
    const int64_t X = wxy[2 * k] + x, Y = wxy[2 * k + 1] + y;
    const int64_t cx = floordiv(X, scale) - px0, cy = floordiv(Y, scale) - py0;
    const T m = mask_channel >= 0 ? parent[mask_channel * plane + cy * pw + cx] : (T)1;
    mask_out[idx] = m;
    const bool hole = m < (T)1;
    for (int c = 0; c < pc; ++c) {
      T v = parent[c * plane + cy * pw + cx];
      if (hole) v = (T)noise_value(prefix, X, Y, (uint32_t)c, &slow);
      out[((int64_t)k * pc + c) * per + rem] = v;
    }
  }
}

// =====================================================================
// K9 base maps  (pipeline.py:72-139)
__global__ void procedural_map_kernel(uint64_t prefix, int cell, int64_t x0, int64_t y0, int w,
                                      int h, int channels, float* __restrict__ out) {
  const int64_t total = (int64_t)channels * w * h;
  const int64_t gx0 = floordiv(x0, cell), gy0 = floordiv(y0, cell);
  int slow = 0;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(idx / ((int64_t)w * h));
    const int rem = (int)(idx - (int64_t)c * w * h);
    const int py = rem / w, px = rem - py * w;
    const int64_t X = x0 + px, Y = y0 + py;
    // fx = (xs / cell) - gx0 in float64 (numpy true_divide then subtract)
    const double fx = rsub(rdiv((double)X, (double)cell), (double)gx0);
    const double fy = rsub(rdiv((double)Y, (double)cell), (double)gy0);
    const double ixf = floor(fx), iyf = floor(fy);
    const double tx = rsub(fx, ixf), ty = rsub(fy, iyf);
    const int64_t gx = gx0 + (int64_t)ixf, gy = gy0 + (int64_t)iyf;
    const double v00 = noise_value(prefix, gx, gy, (uint32_t)c, &slow);
    const double v01 = noise_value(prefix, gx + 1, gy, (uint32_t)c, &slow);
    const double v10 = noise_value(prefix, gx, gy + 1, (uint32_t)c, &slow);
    const double v11 = noise_value(prefix, gx + 1, gy + 1, (uint32_t)c, &slow);
    const double omx = rsub(1.0, tx), omy = rsub(1.0, ty);
    const double top = radd(rmul(v00, omx), rmul(v01, tx));
    const double bot = radd(rmul(v10, omx), rmul(v11, tx));
    out[idx] = __double2float_rn(radd(rmul(top, omy), rmul(bot, ty)));
  }
}

__global__ void corrupt_kernel(const float* __restrict__ in, uint64_t prefix, float level,
                               int64_t x0, int64_t y0, int w, int h, float* __restrict__ out) {
  const int64_t total = (int64_t)w * h;
  int slow = 0;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int py = (int)(idx / w), px = (int)(idx - (int64_t)py * w);
    const float z = noise_value(prefix, x0 + px, y0 + py, 0u, &slow);
    out[idx] = radd(in[idx], rmul(level, z));
  }
}

__global__ void raster_map_kernel(const float* __restrict__ raster, int rc, int rh, int rw,
                                  int mode, int64_t x0, int64_t y0, int w, int h, int channels,
                                  float* __restrict__ out) {
  const int64_t total = (int64_t)channels * w * h;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(idx / ((int64_t)w * h));
    const int rem = (int)(idx - (int64_t)c * w * h);
    const int py = rem / w, px = rem - py * w;
    int64_t X = x0 + px, Y = y0 + py;
    if (mode == 0) {
      X = X < 0 ? 0 : (X > rw - 1 ? rw - 1 : X);
      Y = Y < 0 ? 0 : (Y > rh - 1 ? rh - 1 : Y);
    } else {
      X = pymod(X, rw);
      Y = pymod(Y, rh);
    }
    out[idx] = raster[((int64_t)c * rh + Y) * rw + X];
  }
}

// element-type dispatch for the dtype-generic transforms: calls f(T{}) with
// the C++ type of an IG_DTYPE_* code; returns false for an unknown code
template <typename F>
static bool with_dtype(int32_t dtype, F&& f) {
  switch (dtype) {
    case IG_DTYPE_F32: f(float{}); return true;
    case IG_DTYPE_F64: f(double{}); return true;
    case IG_DTYPE_F16: f(__half{}); return true;
    case IG_DTYPE_I32: f(int32_t{}); return true;
    case IG_DTYPE_I64: f(int64_t{}); return true;
    default: return false;
  }
}


// ---------------------------------------------------------------------
// render normalisation (transforms.py:117-135 normalize_heightmap_u8): per
// image min / max (exact in any order; doubles mapped to order-preserving
// 64-bit keys for the atomics), then ((x - mid) / range + 0.5) * 255 clipped,
// rounded half-to-even (rint) and replicated to 3 channels -- every step an
// IEEE f64 operation, so the bytes equal numpy's
__device__ __forceinline__ unsigned long long f64_key(double v) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double f64_unkey(unsigned long long k) {
  return __longlong_as_double((long long)((k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k));
}
__global__ void minmax_init_kernel(unsigned long long* mm, int b) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < b) { mm[2 * i] = ~0ull; mm[2 * i + 1] = 0ull; }
}
template <typename T>
__global__ void __launch_bounds__(256) minmax_kernel(const T* __restrict__ in, int64_t hw,
                                                     unsigned long long* __restrict__ mm) {
  const int img = blockIdx.y;
  const T* p = in + (int64_t)img * hw;
  double lo = INFINITY, hi = -INFINITY;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < hw;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double v = (double)p[i];
    lo = fmin(lo, v);
    hi = fmax(hi, v);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&mm[2 * img], f64_key(lo));
    atomicMax(&mm[2 * img + 1], f64_key(hi));
  }
}
template <typename T>
__global__ void __launch_bounds__(256) normalize_u8_kernel(const T* __restrict__ in, int64_t hw,
                                                           const unsigned long long* __restrict__ mm,
                                                           uint8_t* __restrict__ out) {
  const int img = blockIdx.y;
  const double mn = f64_unkey(mm[2 * img]), mx = f64_unkey(mm[2 * img + 1]);
  const double rng = fmax(rsub(mx, mn), 255.0);
  const double mid = rdiv(radd(mn, mx), 2.0);
  const T* p = in + (int64_t)img * hw;
  uint8_t* o = out + (int64_t)img * 3 * hw;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < hw;
       i += (int64_t)gridDim.x * blockDim.x) {
    double v = rmul(radd(rdiv(rsub((double)p[i], mid), rng), 0.5), 255.0);
    v = fmin(fmax(v, 0.0), 255.0);
    const uint8_t u = (uint8_t)rint(v);
    o[i] = u;
    o[hw + i] = u;
    o[2 * hw + i] = u;
  }
}
// Horn 3x3 hillshade to uint8 (reference cli.py:230-249): edge-clamped
// neighbours, the gradient sums in the reference's association order, every
// arithmetic step an explicit round-to-nearest float64 op (no FMA contraction
// -- numpy evaluates each product and sum separately), CUDA's float64
// atan / hypot / atan2 / sin / cos for numpy's, round half to even, clamp.
// cz / sz: numpy's cos / sin of the zenith, azi the light's azimuth (radians),
// computed on the host exactly as the reference does.
template <typename T>
__global__ void __launch_bounds__(256) hillshade_u8_kernel(const T* __restrict__ z, int h, int w,
                                                           double cz, double sz, double azi,
                                                           uint8_t* __restrict__ out) {
  const int64_t total = (int64_t)h * w;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int y = (int)(i / w), x = (int)(i - (int64_t)(i / w) * w);
    const int ym = y > 0 ? y - 1 : 0, yp = y < h - 1 ? y + 1 : h - 1;
    const int xm = x > 0 ? x - 1 : 0, xp = x < w - 1 ? x + 1 : w - 1;
    auto at = [&](int yy, int xx) { return (double)z[(int64_t)yy * w + xx]; };
    const double a = at(ym, xm), b = at(ym, x), c = at(ym, xp);
    const double d = at(y, xm), f = at(y, xp);
    const double g = at(yp, xm), hh = at(yp, x), k = at(yp, xp);
    const double right = radd(radd(c, rmul(2.0, f)), k), left = radd(radd(a, rmul(2.0, d)), g);
    const double below = radd(radd(g, rmul(2.0, hh)), k), above = radd(radd(a, rmul(2.0, b)), c);
    const double gx = rdiv(rsub(right, left), 8.0), gy = rdiv(rsub(below, above), 8.0);
    const double slope = atan(hypot(gx, gy));
    const double aspect = atan2(gy, -gx);
    const double lum =
        rmul(255.0, radd(rmul(cz, cos(slope)), rmul(rmul(sz, sin(slope)), cos(rsub(azi, aspect)))));
    const double r = fmin(fmax(rint(lum), 0.0), 255.0);
    out[i] = (uint8_t)r;
  }
}
}  // namespace ig

// =====================================================================
// C-ABI
using namespace ig;

extern "C" {

const char* ig_last_error(void) { return g_err; }
int ig_abi_version(void) { return 1; }
long long ig_launch_count(void) { return g_launches.load(); }

int ig_noise_region(uint64_t seed, uint32_t stream, int64_t x0, int64_t y0, int32_t width,
                    int32_t height, int32_t ch0, int32_t nch, int32_t out_dtype, void* out,
                    int32_t* slow_count, void* cuda_stream) {
  IG_REQUIRE(width > 0 && height > 0 && nch > 0, "noise_region: empty region %dx%dx%d", nch,
             height, width);
  IG_REQUIRE(out != nullptr, "noise_region: null output");
  const uint64_t prefix = noise_prefix(seed, stream);
  const int64_t quads = (int64_t)((width + 3) / 4) * height * nch;
  const int grid = grid_for(quads, 256, 32);
  if (out_dtype == IG_DTYPE_F32)
    { noise_region_kernel<float><<<grid, 256, 0, as_stream(cuda_stream)>>>(
        prefix, x0, y0, width, height, ch0, nch, (float*)out, slow_count); note_launch(); }
  else
    { noise_region_kernel<double><<<grid, 256, 0, as_stream(cuda_stream)>>>(
        prefix, x0, y0, width, height, ch0, nch, (double*)out, slow_count); note_launch(); }
  return cuda_check("ig_noise_region");
}

int ig_phi_analytic(int32_t kind, int32_t radius, double lam, int32_t dtype, const void* src,
                    int32_t src_batched, int64_t src_x0, int64_t src_y0, int32_t src_w,
                    int32_t src_h, int32_t channels, const int64_t* wxy, int32_t n,
                    int32_t window, const void* cond_parent, int64_t cond_x0, int64_t cond_y0,
                    int32_t cond_w, int32_t cond_h, int32_t cond_c, int32_t cond_scale,
                    int32_t cond_mask_channel, uint64_t cond_seed, int32_t cond_fill, void* out,
                    void* cuda_stream) {
  IG_REQUIRE(kind >= 0 && kind <= 2, "phi: unknown kind %d", kind);
  IG_REQUIRE(radius >= 0, "phi: radius must be >= 0");
  IG_REQUIRE(n >= 0 && window > 0 && channels > 0, "phi: bad batch");
  if (n == 0) return IG_OK;
  SrcView s{src, src_batched, src_x0, src_y0, src_w, src_h, channels};
  CondView c{cond_parent, cond_x0, cond_y0, cond_w, cond_h, cond_c, cond_scale < 1 ? 1 : cond_scale,
             cond_mask_channel, cond_fill, noise_prefix(cond_seed, 101u)};
  const int lam_zero = (lam == 0.0);
  // tiled path: bands of up to 16 rows whose staged rows fit 48 KB of SMEM
  {
    const int r = (kind == IG_PHI_IDENTITY || lam_zero) ? 0 : radius;
    const size_t es = dtype == IG_DTYPE_F32 ? 4 : 8;
    int band = 16;
    while (band > 1 && (size_t)(2 * band + 2 * r) * window * es > 48 * 1024) band /= 2;
    const size_t smem = (size_t)(2 * band + 2 * r) * window * es;
    if (smem <= 48 * 1024 && (int64_t)n * channels <= 65535) {
      const dim3 grid((unsigned)((window + band - 1) / band), (unsigned)(n * channels));
      cudaStream_t st = as_stream(cuda_stream);
#define IG_PHI_TILE(T, R, A, B, O)                                                              \
  phi_tile_kernel<T, R><<<grid, 256, smem, st>>>(kind, radius, A, B, lam_zero, s, wxy, window, \
                                                 band, c, (T*)out)
      if (dtype == IG_DTYPE_F32) {
        const float A = (float)(1.0 - lam), B = (float)lam;
        if (r == 0) IG_PHI_TILE(float, 0, A, B, out);
        else if (r == 1) IG_PHI_TILE(float, 1, A, B, out);
        else IG_PHI_TILE(float, -1, A, B, out);
      } else {
        const double A = 1.0 - lam, B = lam;
        if (r == 0) IG_PHI_TILE(double, 0, A, B, out);
        else if (r == 1) IG_PHI_TILE(double, 1, A, B, out);
        else IG_PHI_TILE(double, -1, A, B, out);
      }
#undef IG_PHI_TILE
      note_launch();
      return cuda_check("ig_phi_analytic");
    }
  }
  const int64_t total = (int64_t)n * channels * window * window;
  const int grid = grid_for(total, 256);
  if (dtype == IG_DTYPE_F32)
    { phi_analytic_kernel<float><<<grid, 256, 0, as_stream(cuda_stream)>>>(
        kind, radius, (float)(1.0 - lam), (float)lam, lam_zero, s, wxy, n, window, c,
        (float*)out); note_launch(); }
  else
    { phi_analytic_kernel<double><<<grid, 256, 0, as_stream(cuda_stream)>>>(
        kind, radius, 1.0 - lam, lam, lam_zero, s, wxy, n, window, c, (double*)out); note_launch(); }
  return cuda_check("ig_phi_analytic");
}

int ig_blend(const void* const* win_data, int64_t i0, int64_t j0, int32_t ni, int32_t nj,
             int32_t window, int32_t stride, int64_t off_x, int64_t off_y, int32_t channels,
             int32_t mode, const void* weight, int64_t rx0, int64_t ry0, int32_t rw, int32_t rh,
             int32_t divide, int32_t dtype, void* out, void* cuda_stream) {
  IG_REQUIRE(rw > 0 && rh > 0, "blend: empty region");
  IG_REQUIRE(stride >= 1 && stride <= window, "blend: bad layout");
  IG_REQUIRE(mode == 0 || mode == 1, "blend: bad mode");
  IG_REQUIRE(!(divide && mode == 0), "blend: divide needs weighted mode");
  IG_REQUIRE(mode == 0 || weight != nullptr, "blend: weighted mode needs a weight table");
  // cell fast path: window == 2 * stride, weighted, <= 4 channels, stride % 4 == 0,
  // 16-byte aligned window rows; whole passes of (256 / (stride/4)) rows per cell
  // (2 passes when T * C <= 8 bytes)
  if (mode == 1 && window == 2 * stride && channels >= 1 && channels <= 4 && stride % 4 == 0 &&
      256 % (stride / 4) == 0) {
    const int es = dtype == IG_DTYPE_F32 ? 4 : 8;
    const int passes = es * channels <= 8 ? 2 : 1;
    const int64_t ci_lo = floordiv(rx0 - off_x, stride), ci_hi = floordiv(rx0 + rw - 1 - off_x, stride);
    const int64_t cj_lo = floordiv(ry0 - off_y, stride), cj_hi = floordiv(ry0 + rh - 1 - off_y, stride);
    const int ncx = (int)(ci_hi - ci_lo + 1), ncy = (int)(cj_hi - cj_lo + 1);
    const int rows_per_cta = passes * (256 / (stride / 4));
    const int64_t cells = (int64_t)ncx * ncy;
    if (stride % rows_per_cta == 0 && cells * (stride / rows_per_cta) < (1ll << 31)) {
      cudaStream_t st = as_stream(cuda_stream);
#define IG_BLEND_CELLS(T, C)                                                                   \
  launch_blend_cells<T, C>(win_data, i0, j0, ni, nj, window, stride, off_x, off_y, weight, rx0, \
                           ry0, rw, rh, divide, ci_lo, cj_lo, ncx, cells, out, st)
      if (dtype == IG_DTYPE_F32) {
        switch (channels) {
          case 1: IG_BLEND_CELLS(float, 1); break;
          case 2: IG_BLEND_CELLS(float, 2); break;
          case 3: IG_BLEND_CELLS(float, 3); break;
          default: IG_BLEND_CELLS(float, 4); break;
        }
      } else {
        switch (channels) {
          case 1: IG_BLEND_CELLS(double, 1); break;
          case 2: IG_BLEND_CELLS(double, 2); break;
          case 3: IG_BLEND_CELLS(double, 3); break;
          default: IG_BLEND_CELLS(double, 4); break;
        }
      }
#undef IG_BLEND_CELLS
      return cuda_check("ig_blend");
    }
  }
  const dim3 grid((unsigned)((rw + 1023) / 1024), (unsigned)(rh < 65535 ? rh : 65535));
  if (dtype == IG_DTYPE_F32)
    { blend_kernel<float><<<grid, 256, 0, as_stream(cuda_stream)>>>(
        (const float* const*)win_data, i0, j0, ni, nj, window, stride, off_x, off_y, channels,
        mode, (const float*)weight, rx0, ry0, rw, rh, divide, (float*)out); note_launch(); }
  else
    { blend_kernel<double><<<grid, 256, 0, as_stream(cuda_stream)>>>(
        (const double* const*)win_data, i0, j0, ni, nj, window, stride, off_x, off_y, channels,
        mode, (const double*)weight, rx0, ry0, rw, rh, divide, (double*)out); note_launch(); }
  return cuda_check("ig_blend");
}

int ig_divide_weighted(const void* raw, int32_t channels, int64_t npix, int32_t dtype, void* out,
                       void* cuda_stream) {
  if (npix <= 0) return IG_OK;
  const int grid = grid_for(npix, 256);
  if (dtype == IG_DTYPE_F32)
    { divide_weighted_kernel<float><<<grid, 256, 0, as_stream(cuda_stream)>>>(
        (const float*)raw, channels, npix, (float*)out); note_launch(); }
  else
    { divide_weighted_kernel<double><<<grid, 256, 0, as_stream(cuda_stream)>>>(
        (const double*)raw, channels, npix, (double*)out); note_launch(); }
  return cuda_check("ig_divide_weighted");
}

int ig_box_mean(const void* in, int32_t planes, int32_t h, int32_t w, int32_t radius,
                int32_t dtype, void* out, void* cuda_stream) {
  IG_REQUIRE(radius >= 0, "radius must be >= 0");
  const int64_t total = (int64_t)planes * h * w;
  if (total == 0) return IG_OK;
  const int grid = grid_for(total, 256);
  if (dtype == IG_DTYPE_F32)
    { box_mean_kernel<float><<<grid, 256, 0, as_stream(cuda_stream)>>>((const float*)in, planes, h,
                                                                     w, radius, (float*)out); note_launch(); }
  else
    { box_mean_kernel<double><<<grid, 256, 0, as_stream(cuda_stream)>>>(
        (const double*)in, planes, h, w, radius, (double*)out); note_launch(); }
  return cuda_check("ig_box_mean");
}

int ig_blur_block_mean_f64(const void* in, int32_t in_dtype, int32_t planes, int32_t h, int32_t w,
                           int32_t blur_iters, int32_t factor, double* scratch, double* low,
                           void* cuda_stream) {
  IG_REQUIRE(factor >= 1 && h % factor == 0 && w % factor == 0,
             "spatial dims %dx%d not divisible by factor %d", h, w, factor);
  const int64_t total = (int64_t)planes * h * w;
  cudaStream_t st = as_stream(cuda_stream);
  if (total == 0) return IG_OK;
  // fused single-pass path (blur_iters <= 1)
  if (blur_iters <= 1 && planes <= 65535) {
    const int r = blur_iters;
    const int TH = factor * ((16 + factor - 1) / factor), TW = factor * ((128 + factor - 1) / factor);
    const size_t smem = ((size_t)(TH + 2 * r) * (TW + 2 * r) + (size_t)TH * (TW + 2 * r)) * 8;
    if (smem <= 48 * 1024) {
      const dim3 grid((unsigned)((w + TW - 1) / TW), (unsigned)((h + TH - 1) / TH), (unsigned)planes);
      if (in_dtype == IG_DTYPE_F32)
        { blur_block_mean_tile_kernel<float><<<grid, 256, smem, st>>>((const float*)in, h, w, r,
                                                                      factor, TH, TW, low); note_launch(); }
      else
        { blur_block_mean_tile_kernel<double><<<grid, 256, smem, st>>>((const double*)in, h, w, r,
                                                                       factor, TH, TW, low); note_launch(); }
      return cuda_check("ig_blur_block_mean_f64");
    }
  }
  const int grid = grid_for(total, 256);
  double* a = scratch;
  double* b = scratch + total;
  if (in_dtype == IG_DTYPE_F32)
    { widen_kernel<float><<<grid, 256, 0, st>>>((const float*)in, total, a); note_launch(); }
  else
    { widen_kernel<double><<<grid, 256, 0, st>>>((const double*)in, total, a); note_launch(); }
  for (int it = 0; it < blur_iters; ++it) {
    { box_mean_kernel<double><<<grid, 256, 0, st>>>(a, planes, h, w, 1, b); note_launch(); }
    double* t = a; a = b; b = t;
  }
  const int64_t lt = total / ((int64_t)factor * factor);
  { block_mean_kernel<double><<<grid_for(lt, 256), 256, 0, st>>>(a, planes, h, w, factor, low); note_launch(); }
  return cuda_check("ig_blur_block_mean_f64");
}

int ig_laplacian_residual(const void* x, int32_t x_dtype, const double* low, int32_t planes,
                          int32_t h, int32_t w, int32_t factor, double* high, void* cuda_stream) {
  if ((int64_t)planes * h * w == 0) return IG_OK;
  {
    const dim3 grid((unsigned)((w + 1023) / 1024),
                    (unsigned)((int64_t)planes * h < 65535 ? (int64_t)planes * h : 65535));
    if (x_dtype == IG_DTYPE_F32)
      { laplacian_residual_rows_kernel<float><<<grid, 256, 0, as_stream(cuda_stream)>>>(
          (const float*)x, low, planes, h, w, factor, high); note_launch(); }
    else
      { laplacian_residual_rows_kernel<double><<<grid, 256, 0, as_stream(cuda_stream)>>>(
          (const double*)x, low, planes, h, w, factor, high); note_launch(); }
    return cuda_check("ig_laplacian_residual");
  }
}

int ig_laplacian_merge(const double* low, const double* high, int32_t planes, int32_t h,
                       int32_t w, int32_t factor, int32_t out_dtype, int32_t square_out,
                       void* out, void* cuda_stream) {
  IG_REQUIRE(!square_out || out_dtype == IG_DTYPE_F32 || out_dtype == IG_DTYPE_F64,
             "laplacian_merge: signed-square output needs a float32/float64 dtype");
  if ((int64_t)planes * h * w == 0) return IG_OK;
  const dim3 grid((unsigned)((w + 1023) / 1024),
                  (unsigned)((int64_t)planes * h < 65535 ? (int64_t)planes * h : 65535));
  const bool ok = with_dtype(out_dtype, [&](auto tag) {
    using TO = decltype(tag);
    laplacian_merge_rows_kernel<TO><<<grid, 256, 0, as_stream(cuda_stream)>>>(
        low, high, planes, h, w, factor, square_out, (TO*)out);
    note_launch();
  });
  IG_REQUIRE(ok, "laplacian_merge: unknown dtype %d", out_dtype);
  return cuda_check("ig_laplacian_merge");
}

int ig_signed_pow(const void* in, int64_t n, int32_t op, int32_t dtype, void* out,
                  void* cuda_stream) {
  IG_REQUIRE(op == 0 || op == 1, "signed_pow: op must be 0 (sqrt) or 1 (square)");
  if (n <= 0) return IG_OK;
  const int grid = grid_for(n, 256);
  cudaStream_t st = as_stream(cuda_stream);
  if (dtype == IG_DTYPE_F32)
    { signed_pow_kernel<float><<<grid, 256, 0, st>>>((const float*)in, n, op, (float*)out); note_launch(); }
  else if (dtype == IG_DTYPE_F64)
    { signed_pow_kernel<double><<<grid, 256, 0, st>>>((const double*)in, n, op, (double*)out); note_launch(); }
  else if (op == 1 && dtype == IG_DTYPE_I32)
    { signed_square_int_kernel<int32_t><<<grid, 256, 0, st>>>((const int32_t*)in, n, (int32_t*)out); note_launch(); }
  else if (op == 1 && dtype == IG_DTYPE_I64)
    { signed_square_int_kernel<int64_t><<<grid, 256, 0, st>>>((const int64_t*)in, n, (int64_t*)out); note_launch(); }
  else
    IG_REQUIRE(false, "signed_pow: op %d undefined for dtype %d", op, dtype);
  return cuda_check("ig_signed_pow");
}

int ig_block_mean(const void* in, int32_t dtype, int32_t planes, int32_t h, int32_t w,
                  int32_t factor, void* out, void* cuda_stream) {
  IG_REQUIRE(factor >= 1 && h % factor == 0 && w % factor == 0,
             "spatial dims %dx%d not divisible by factor %d", h, w, factor);
  IG_REQUIRE(dtype == IG_DTYPE_F32 || dtype == IG_DTYPE_F64,
             "block_mean: accumulation dtype must be float32 or float64");
  const int64_t lt = (int64_t)planes * (h / factor) * (w / factor);
  if (lt == 0) return IG_OK;
  if (dtype == IG_DTYPE_F32)
    { block_mean_kernel<float><<<grid_for(lt, 256), 256, 0, as_stream(cuda_stream)>>>(
        (const float*)in, planes, h, w, factor, (float*)out); note_launch(); }
  else
    { block_mean_kernel<double><<<grid_for(lt, 256), 256, 0, as_stream(cuda_stream)>>>(
        (const double*)in, planes, h, w, factor, (double*)out); note_launch(); }
  return cuda_check("ig_block_mean");
}

int ig_convert(const void* in, int32_t in_dtype, int64_t n, void* out, int32_t out_dtype,
               void* cuda_stream) {
  if (n <= 0) return IG_OK;
  const int grid = grid_for(n, 256);
  bool ok_out = false;
  const bool ok_in = with_dtype(in_dtype, [&](auto ti) {
    using TI = decltype(ti);
    ok_out = with_dtype(out_dtype, [&](auto to) {
      using TO = decltype(to);
      convert_kernel<TO, TI><<<grid, 256, 0, as_stream(cuda_stream)>>>((const TI*)in, n, (TO*)out);
      note_launch();
    });
  });
  IG_REQUIRE(ok_in && ok_out, "convert: unknown dtype pair %d -> %d", in_dtype, out_dtype);
  return cuda_check("ig_convert");
}

int ig_normalize_u8(const void* in, int32_t dtype, int32_t images, int64_t hw, void* minmax,
                    uint8_t* out, void* cuda_stream) {
  IG_REQUIRE(dtype == IG_DTYPE_F32 || dtype == IG_DTYPE_F64, "normalize_u8: float input");
  if (images <= 0 || hw <= 0) return IG_OK;
  IG_REQUIRE(images <= 65535, "normalize_u8: at most 65535 images per call");
  cudaStream_t st = as_stream(cuda_stream);
  unsigned long long* mm = (unsigned long long*)minmax;
  { minmax_init_kernel<<<(images + 255) / 256, 256, 0, st>>>(mm, images); note_launch(); }
  const int bx = grid_for(hw, 256, 4 > images ? 4 : 1);
  const dim3 grid((unsigned)bx, (unsigned)images);
  if (dtype == IG_DTYPE_F32) {
    minmax_kernel<float><<<grid, 256, 0, st>>>((const float*)in, hw, mm); note_launch();
    normalize_u8_kernel<float><<<grid, 256, 0, st>>>((const float*)in, hw, mm, out); note_launch();
  } else {
    minmax_kernel<double><<<grid, 256, 0, st>>>((const double*)in, hw, mm); note_launch();
    normalize_u8_kernel<double><<<grid, 256, 0, st>>>((const double*)in, hw, mm, out); note_launch();
  }
  return cuda_check("ig_normalize_u8");
}

int ig_hillshade_u8(const void* elev, int32_t dtype, int32_t h, int32_t w, double cos_zenith,
                    double sin_zenith, double azimuth, uint8_t* out, void* cuda_stream) {
  IG_REQUIRE(dtype == IG_DTYPE_F32 || dtype == IG_DTYPE_F64, "hillshade_u8: float input");
  IG_REQUIRE(h >= 0 && w >= 0, "hillshade_u8: negative shape %dx%d", h, w);
  if (h == 0 || w == 0) return IG_OK;
  const int grid = grid_for((int64_t)h * w, 256);
  if (dtype == IG_DTYPE_F32)
    { hillshade_u8_kernel<float><<<grid, 256, 0, as_stream(cuda_stream)>>>(
        (const float*)elev, h, w, cos_zenith, sin_zenith, azimuth, out); note_launch(); }
  else
    { hillshade_u8_kernel<double><<<grid, 256, 0, as_stream(cuda_stream)>>>(
        (const double*)elev, h, w, cos_zenith, sin_zenith, azimuth, out); note_launch(); }
  return cuda_check("ig_hillshade_u8");
}

int ig_upsample_nn(const void* in, int32_t elem_bytes, int64_t planes, int32_t h, int32_t w,
                   int32_t factor, void* out, void* cuda_stream) {
  IG_REQUIRE(factor >= 1, "upsample_nn: factor must be >= 1");
  const int64_t total = planes * h * factor * (int64_t)w * factor;
  if (total == 0) return IG_OK;
  const int grid = grid_for(total, 256);
  cudaStream_t st = as_stream(cuda_stream);
  switch (elem_bytes) {
    case 1: upsample_nn_kernel<uint8_t><<<grid, 256, 0, st>>>((const uint8_t*)in, planes, h, w, factor, (uint8_t*)out); break;
    case 2: upsample_nn_kernel<uint16_t><<<grid, 256, 0, st>>>((const uint16_t*)in, planes, h, w, factor, (uint16_t*)out); break;
    case 4: upsample_nn_kernel<uint32_t><<<grid, 256, 0, st>>>((const uint32_t*)in, planes, h, w, factor, (uint32_t*)out); break;
    case 8: upsample_nn_kernel<uint64_t><<<grid, 256, 0, st>>>((const uint64_t*)in, planes, h, w, factor, (uint64_t*)out); break;
    default: IG_REQUIRE(false, "upsample_nn: element size %d", elem_bytes);
  }
  note_launch();
  return cuda_check("ig_upsample_nn");
}

int ig_patch_features(const void* in, int64_t tile_stride, int32_t n, int32_t h, int32_t w,
                      int32_t patch, int32_t rank, int32_t dtype, void* out, void* cuda_stream) {
  IG_REQUIRE(patch >= 1 && h % patch == 0 && w % patch == 0,
             "region %dx%d not divisible by patch size %d", h, w, patch);
  IG_REQUIRE(rank >= 1 && rank <= patch * patch, "bad percentile rank %d", rank);
  const int64_t total = (int64_t)n * (h / patch) * (w / patch);
  if (total == 0) return IG_OK;
  const int grid = grid_for(total, 128);
  if (dtype == IG_DTYPE_F32)
    { patch_features_kernel<float><<<grid, 128, 0, as_stream(cuda_stream)>>>(
        (const float*)in, tile_stride, n, h, w, patch, rank, (float*)out); note_launch(); }
  else
    { patch_features_kernel<double><<<grid, 128, 0, as_stream(cuda_stream)>>>(
        (const double*)in, tile_stride, n, h, w, patch, rank, (double*)out); note_launch(); }
  return cuda_check("ig_patch_features");
}

int ig_condition_window(const void* parent, int64_t px0, int64_t py0, int32_t pw, int32_t ph,
                        int32_t pc, int32_t scale, int32_t mask_channel, uint64_t seed,
                        const int64_t* wxy, int32_t n, int32_t window, int32_t dtype, void* out,
                        void* mask_out, void* cuda_stream) {
  IG_REQUIRE(scale >= 1, "conditioning scale must be >= 1");
  if (n == 0) return IG_OK;
  const uint64_t prefix = noise_prefix(seed, 101u);
  const int grid = grid_for((int64_t)n * window * window, 256);
  if (dtype == IG_DTYPE_F32)
    { condition_window_kernel<float><<<grid, 256, 0, as_stream(cuda_stream)>>>(
        (const float*)parent, px0, py0, pw, ph, pc, scale, mask_channel, prefix, wxy, n, window,
        (float*)out, (float*)mask_out); note_launch(); }
  else
    { condition_window_kernel<double><<<grid, 256, 0, as_stream(cuda_stream)>>>(
        (const double*)parent, px0, py0, pw, ph, pc, scale, mask_channel, prefix, wxy, n, window,
        (double*)out, (double*)mask_out); note_launch(); }
  return cuda_check("ig_condition_window");
}

int ig_procedural_map(uint64_t seed, uint32_t stream, int32_t cell, int64_t x0, int64_t y0,
                      int32_t w, int32_t h, int32_t channels, float* out, void* cuda_stream) {
  IG_REQUIRE(cell >= 1, "cell must be >= 1");
  const int64_t total = (int64_t)channels * w * h;
  if (total == 0) return IG_OK;
  { procedural_map_kernel<<<grid_for(total, 256), 256, 0, as_stream(cuda_stream)>>>(
      noise_prefix(seed, stream), cell, x0, y0, w, h, channels, out); note_launch(); }
  return cuda_check("ig_procedural_map");
}

int ig_corrupt(const float* in, const double* levels_host, int32_t channels, uint64_t seed,
               int64_t x0, int64_t y0, int32_t w, int32_t h, float* out, void* cuda_stream) {
  cudaStream_t st = as_stream(cuda_stream);
  const int64_t plane = (int64_t)w * h;
  for (int c = 0; c < channels; ++c) {
    const double lv = levels_host[c];
    IG_REQUIRE(lv >= 0.0, "corruption noise levels must be >= 0");
    if (lv == 0.0) {
      if (out != in)
        cudaMemcpyAsync(out + c * plane, in + c * plane, plane * sizeof(float),
                        cudaMemcpyDeviceToDevice, st);
      continue;
    }
    { corrupt_kernel<<<grid_for(plane, 256), 256, 0, st>>>(
        in + c * plane, noise_prefix(seed, 201u + (uint32_t)c), (float)lv, x0, y0, w, h,
        out + c * plane); note_launch(); }
  }
  return cuda_check("ig_corrupt");
}

int ig_raster_map(const float* raster, int32_t rc, int32_t rh, int32_t rw, int32_t mode,
                  int64_t x0, int64_t y0, int32_t w, int32_t h, int32_t channels, float* out,
                  void* cuda_stream) {
  IG_REQUIRE(channels <= rc, "user map has %d channels, %d requested", rc, channels);
  const int64_t total = (int64_t)channels * w * h;
  if (total == 0) return IG_OK;
  { raster_map_kernel<<<grid_for(total, 256), 256, 0, as_stream(cuda_stream)>>>(
      raster, rc, rh, rw, mode, x0, y0, w, h, channels, out); note_launch(); }
  return cuda_check("ig_raster_map");
}

// ---------------------------------------------------------------------------
// Peer-memory halo exchange: a rank exports the device
// allocation holding its Phi windows as a CUDA IPC handle; a neighbour maps it
// (peer access enabled lazily from ITS current device, so its blend kernel
// reads the windows straight over NVLink -- the "exchange" is the blend's own
// loads, no send/recv copy).  Handles refer to the whole allocation, so the
// window's byte offset inside it travels alongside.
int ig_ipc_export(const void* dev_ptr, uint8_t* handle64, int64_t* offset) {
  IG_REQUIRE(dev_ptr != nullptr && handle64 != nullptr && offset != nullptr,
             "ipc_export: null argument");
  // driver entry point fetched at run time (no link-time libcuda dependency:
  // the library must load on a host without a driver)
  using AddrRangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  static AddrRangeFn addr_range = nullptr;
  if (!addr_range) {
    cudaDriverEntryPointQueryResult q;
    void* fp = nullptr;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fp, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      set_error("ipc_export: cuMemGetAddressRange unavailable");
      return IG_ERR_CUDA;
    }
    addr_range = reinterpret_cast<AddrRangeFn>(fp);
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (addr_range(&base, &size, (CUdeviceptr)dev_ptr) != CUDA_SUCCESS) {
    set_error("ipc_export: pointer %p is not a device allocation", dev_ptr);
    return IG_ERR_ARG;
  }
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
  if (e != cudaSuccess) {
    set_error("ipc_export: cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
    return IG_ERR_CUDA;
  }
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  memcpy(handle64, &h, 64);
  *offset = (int64_t)((CUdeviceptr)dev_ptr - base);
  return IG_OK;
}

int ig_ipc_open(const uint8_t* handle64, void** base_out) {
  IG_REQUIRE(handle64 != nullptr && base_out != nullptr, "ipc_open: null argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, 64);
  cudaError_t e = cudaIpcOpenMemHandle(base_out, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) {
    set_error("ipc_open: cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
    return IG_ERR_CUDA;
  }
  return IG_OK;
}

// Dedicated exchange allocation (outside any caching allocator): an IPC handle
// maps the WHOLE allocation containing a pointer, so exporting a window that
// lives inside a multi-GB pool segment would map the pool on every peer.
int ig_ipc_alloc(int64_t bytes, void** ptr_out) {
  IG_REQUIRE(bytes > 0 && ptr_out != nullptr, "ipc_alloc: bad size");
  cudaError_t e = cudaMalloc(ptr_out, (size_t)bytes);
  if (e != cudaSuccess) {
    set_error("ipc_alloc: cudaMalloc(%lld): %s", (long long)bytes, cudaGetErrorString(e));
    return IG_ERR_CUDA;
  }
  return IG_OK;
}

int ig_ipc_free(void* ptr) {
  cudaError_t e = cudaFree(ptr);
  if (e != cudaSuccess) {
    set_error("ipc_free: %s", cudaGetErrorString(e));
    return IG_ERR_CUDA;
  }
  return IG_OK;
}

int ig_ipc_close(void* base) {
  cudaError_t e = cudaIpcCloseMemHandle(base);
  if (e != cudaSuccess) {
    set_error("ipc_close: cudaIpcCloseMemHandle: %s", cudaGetErrorString(e));
    return IG_ERR_CUDA;
  }
  return IG_OK;
}

}  // extern "C"
