// INDIRECT tile cache on the device (store.py:358-426 _finalized_mask,
// _gather_tiles, _commit_region).
//
// The reference keeps, per tensor, a dict of (C, ts, ts) numpy tiles plus a
// bool "finalized" mask per tile; a read blends the windows touching
// not-yet-finalized pixels, overwrites the finalized pixels with their
// committed tile values, and commits the whole region back.  Here every tile
// and its mask (one byte per pixel) live in HBM and ONE launch does the
// overlay and the commit: per pixel of the region, a finalized pixel copies
// tile -> out, any other pixel copies out -> tile and marks itself finalized.
// That equals gather-then-commit because committing a finalized pixel writes
// back the value it was just gathered from.  The host keeps its own copy of
// the masks for control flow (which windows need regeneration) only.
#include "ig_common.cuh"

namespace ig {

// tile table: for the tile box [tx0, tx0 + ntx) x [ty0, ty0 + nty), entry
// 2*(ty*ntx + tx) is the tile's data pointer, +1 its mask pointer
template <typename E>
__global__ void __launch_bounds__(256) tiles_resolve_kernel(
    const int64_t* __restrict__ table, int64_t tx0, int64_t ty0, int ntx, int ts_log2,
    int channels, int64_t rx0, int64_t ry0, int rw, int rh, E* __restrict__ out) {
  const int ts = 1 << ts_log2;
  const int64_t npix = (int64_t)rw * rh;
  const int64_t plane = npix;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < npix;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int y = (int)(p / rw), x = (int)(p - (int64_t)y * rw);
    const int64_t X = rx0 + x, Y = ry0 + y;
    // power-of-two tiles: arithmetic shift == Python floor division
    const int64_t tx = X >> ts_log2, ty = Y >> ts_log2;
    const int lx = (int)(X - (tx << ts_log2)), ly = (int)(Y - (ty << ts_log2));
    const int64_t slot = (ty - ty0) * ntx + (tx - tx0);
    E* tile = reinterpret_cast<E*>(table[2 * slot]);
    uint8_t* mask = reinterpret_cast<uint8_t*>(table[2 * slot + 1]);
    const int64_t tp = (int64_t)ly * ts + lx;
    if (mask[tp]) {
      for (int c = 0; c < channels; ++c) out[c * plane + p] = tile[(int64_t)c * ts * ts + tp];
    } else {
      for (int c = 0; c < channels; ++c) tile[(int64_t)c * ts * ts + tp] = out[c * plane + p];
      mask[tp] = 1;
    }
  }
}

}  // namespace ig

using namespace ig;

extern "C" int ig_tiles_resolve(const int64_t* table, int64_t tx0, int64_t ty0, int32_t ntx,
                                int32_t nty, int32_t tile_size, int32_t channels,
                                int32_t elem_bytes, int64_t rx0, int64_t ry0, int32_t rw,
                                int32_t rh, void* out, void* cuda_stream) {
  IG_REQUIRE(tile_size > 0 && (tile_size & (tile_size - 1)) == 0,
             "tiles: tile size must be a power of two, got %d", tile_size);
  IG_REQUIRE(ntx > 0 && nty > 0 && channels > 0, "tiles: empty tile box");
  IG_REQUIRE(floordiv(rx0, tile_size) == tx0 && floordiv(ry0, tile_size) == ty0,
             "tiles: tile box origin does not contain the region origin");
  IG_REQUIRE(floordiv(rx0 + rw - 1, tile_size) < tx0 + ntx &&
             floordiv(ry0 + rh - 1, tile_size) < ty0 + nty, "tiles: tile box too small");
  const int64_t npix = (int64_t)rw * rh;
  if (npix <= 0) return IG_OK;
  const int lg = __builtin_ctz((unsigned)tile_size);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(cuda_stream);
  const int grid = grid_for(npix, 256);
  if (elem_bytes == 4)
    tiles_resolve_kernel<float><<<grid, 256, 0, st>>>(table, tx0, ty0, ntx, lg, channels, rx0, ry0,
                                                      rw, rh, (float*)out);
  else if (elem_bytes == 8)
    tiles_resolve_kernel<double><<<grid, 256, 0, st>>>(table, tx0, ty0, ntx, lg, channels, rx0,
                                                       ry0, rw, rh, (double*)out);
  else
    IG_REQUIRE(false, "tiles: element size %d", elem_bytes);
  note_launch();
  return cuda_check("ig_tiles_resolve");
}
