// Field staging through shared-memory bricks for the paired scalar march
// (north star: "the strided, zero-copy field access ... is staged through
// TMA or shared-memory bricks"; reference gather raycast.py:182-199,
// fields.py:274-276).
//
// Same tile schedule, ray setup, guard proof, pair merge and classification
// as march_fast_kernel<1,1,1,LINE,1,0,float> (march.cu), but every warp
// marches its 8x2-ray tile in chunks of ISC_STAGE_CHUNK station pairs: the
// cell indices of a ray are monotone in k on every axis, so the box of base
// cells a chunk touches is spanned by the chunk's first and last stations of
// each lane; the warp reduces it, copies the box (+1 corner on each axis)
// row by row from the zero-copy field into its slice of shared memory with
// 4-byte cp.async (any strides, no alignment requirement), and reads the 8
// trilinear corners of each sample from shared memory.  A box larger than
// the warp's slice (far-apart rays, long chunks) falls back to the global
// gather for that chunk.  Values and arithmetic are the fast kernel's, so
// images are bit-identical; only where the corners come from changes.
//
// TMA (cp.async.bulk.tensor) is not used: a tensor map needs 16-byte global
// strides, and a zero-copy guarded field has a (n+2)*4-byte row pitch (4104
// B at 1024^3).  1-D bulk copies need 16-byte aligned, 16-byte multiple
// rows, which a box row of ~10 floats at an arbitrary x is not.
//
// Experiment switch: ISC_STAGE=1 routes the f32 guarded trilinear paired
// march here (DESIGN.md §4 records the measured A/B).
#include <climits>
#include <cstdlib>

#include "march_common.cuh"
#include "sample.cuh"

namespace isc {

#ifndef ISC_STAGE_CHUNK
#define ISC_STAGE_CHUNK 8  // station pairs per staged chunk
#endif
#ifndef ISC_STAGE_WARP_FLOATS
#define ISC_STAGE_WARP_FLOATS 1536  // per-warp box capacity (6 KB)
#endif
constexpr int kStageThreads = 256;
constexpr int kStageWarps = kStageThreads / 32;

__device__ __forceinline__ void cp_async4(float* dst_smem, const float* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst_smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Trilinear sample from the staged box: identical operations to fast_sample.
__device__ __forceinline__ float box_sample(const float* box, int ex, int exy, int bx, int by, int bz,
                                            const double p[3]) {
  int ix, iy, iz;
  const double flx = floor_split(p[0], ix), fly = floor_split(p[1], iy), flz = floor_split(p[2], iz);
  const float fx = (float)dsub(p[0], flx), fy = (float)dsub(p[1], fly), fz = (float)dsub(p[2], flz);
  const float* b = box + ((iz - bz) * exy + (iy - by) * ex + (ix - bx));
  const float v000 = b[0], v100 = b[1], v010 = b[ex], v110 = b[ex + 1];
  const float* c = b + exy;
  const float v001 = c[0], v101 = c[1], v011 = c[ex], v111 = c[ex + 1];
  const float a0 = fmaf(fx, v100 - v000, v000), a1 = fmaf(fx, v110 - v010, v010);
  const float a2 = fmaf(fx, v101 - v001, v001), a3 = fmaf(fx, v111 - v011, v011);
  const float b0 = fmaf(fy, a1 - a0, a0), b1 = fmaf(fy, a3 - a2, a2);
  return fmaf(fz, b1 - b0, b0);
}

template <int LINE>
__global__ void __launch_bounds__(kStageThreads, 4)
    march_staged_kernel(const __grid_constant__ isc_render_args a, const FastField F, int tiles_x, int tiles_y,
                        int super_x, int n_codes, int tw_log2, int tile_x0, int tile_y0) {
  extern __shared__ float4 smem4[];
  float* lut_s = reinterpret_cast<float*>(smem4);  // planar LUT (LINE == 0 only), then the warps' boxes
  float* boxes = reinterpret_cast<float*>(smem4 + (LINE == 0 ? ISC_LUT_ENTRIES : 0));
  if (LINE == 0) {
    lut_fill(lut_s, reinterpret_cast<const float4*>(a.src[0].lut));
    __syncthreads();
  }
  const int lane = threadIdx.x & 31;
  float* box = boxes + (threadIdx.x >> 5) * ISC_STAGE_WARP_FLOATS;
  const float* __restrict__ fld = reinterpret_cast<const float*>(F.f);
  const isc_source& s = a.src[0];
  const float lo = s.range_lo, inv = 1.0f / (s.range_hi - s.range_lo);
  const double* o = a.camera.origin;
  const double step = a.step;
  uint32_t* err = a.error_word;
  unsigned long long warp_stations = 0;
  const int tw = 1 << tw_log2, th = 16 >> tw_log2;
  const int q = lane & 15, parity = lane >> 4;

  for (;;) {
    int t = 0;
    if (lane == 0) t = (int)atomicAdd(a.work_counter, 1u);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= n_codes) break;
    const int sblk = t >> 6, w = t & 63;
    int tx = (sblk % super_x) * 8 + morton3(w, 0);
    int ty = (sblk / super_x) * 8 + morton3(w, 1);
    if (tx >= tiles_x || ty >= tiles_y) continue;
    tx += tile_x0;
    ty += tile_y0;
    const int px = tx * tw + (q & (tw - 1)), py = ty * th + (q >> tw_log2);
    const bool in_img = px < a.camera.width && py < a.camera.height;
    Ray r;
    if (in_img) {
      setup_ray(a, px, py, r);
    } else {
      r.hit = false;
      r.k_lo = r.k_hi = 0;
    }
    const long long n = r.hit ? (r.k_hi - r.k_lo) : 0;
    long long nm = n;
    if (n > 0) {  // guard contract proven from the end stations (march_fast_kernel)
      double pa[3], pb[3];
      station_pos(o, r.d, dmul((double)r.k_lo, step), pa);
      station_pos(o, r.d, dmul((double)(r.k_hi - 1), step), pb);
      if (!guard_ok(F, pa) || !guard_ok(F, pb)) {
        if (err && !parity) atomicAdd(err, 1u);
        nm = 0;
      }
    }
    const unsigned trips = __reduce_max_sync(0xffffffffu, (unsigned)((nm + 1) >> 1));
    double kd = (double)(r.k_lo + parity);
    int left = (int)nm - parity;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (unsigned j0 = 0; j0 < trips; j0 += ISC_STAGE_CHUNK) {
      const int jn = (int)min((unsigned)ISC_STAGE_CHUNK, trips - j0);
      // this lane's stations in the chunk: kd, kd+2, ..., kd+2(cnt-1)
      const int cnt = left > 0 ? min(jn, (left + 1) >> 1) : 0;
      int c0[3] = {INT_MAX, INT_MAX, INT_MAX}, c1[3] = {INT_MIN, INT_MIN, INT_MIN};
      if (cnt > 0) {
        double pa[3], pb[3];
        station_pos(o, r.d, dmul(kd, step), pa);
        station_pos(o, r.d, dmul(dadd(kd, 2.0 * (cnt - 1)), step), pb);
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
          int ia, ib;
          floor_split(pa[ax], ia);
          floor_split(pb[ax], ib);
          c0[ax] = min(ia, ib);
          c1[ax] = max(ia, ib);
        }
      }
      int bx = __reduce_min_sync(0xffffffffu, c0[0]), by = __reduce_min_sync(0xffffffffu, c0[1]);
      int bz = __reduce_min_sync(0xffffffffu, c0[2]);
      const int ex = __reduce_max_sync(0xffffffffu, c1[0]) - bx + 2;
      const int ey = __reduce_max_sync(0xffffffffu, c1[1]) - by + 2;
      const int ez = __reduce_max_sync(0xffffffffu, c1[2]) - bz + 2;
      const int exy = ex * ey;
      const bool any = bx != INT_MAX;
      const bool staged = any && ex > 0 && ey > 0 && ez > 0 && exy * ez <= ISC_STAGE_WARP_FLOATS;
      if (staged) {
        const int vol = exy * ez;
        const float inv_ex = 1.0f / (float)ex, inv_exy = 1.0f / (float)exy;
        const float* g0 = fld + ((bz - F.lo[2]) * F.sz + (by - F.lo[1]) * F.sy + (bx - F.lo[0]) * F.sx);
        for (int e = lane; e < vol; e += 32) {
          const int z = (int)(((float)e + 0.5f) * inv_exy);
          const int rem = e - z * exy;
          const int y = (int)(((float)rem + 0.5f) * inv_ex);
          const int x = rem - y * ex;
          cp_async4(box + e, g0 + (z * F.sz + y * F.sy + x * F.sx));
        }
        cp_async_wait_all();
        __syncwarp();
      }
      for (int i = 0; i < jn; ++i, left -= 2, kd = dadd(kd, 2.0)) {
        float4 c = make_float4(0.f, 0.f, 0.f, 0.f);
        if (left > 0) {
          double p0[3];
          station_pos(o, r.d, dmul(kd, step), p0);
          const float v0 = staged ? box_sample(box, ex, exy, bx, by, bz, p0)
                                  : fast_sample<true, true, false, float>(F, p0, err);
          float vv[4] = {v0, 0.f, 0.f, 0.f};
          const float s0 = s.n_steps ? run_chain(s, vv, 1) : v0;
          if constexpr (LINE > 0) c = classify_line_premul<LINE>(s, lo, inv, s0);
          else c = premultiply(classify(lut_s, lo, inv, s0));
        }
        const float4 odd = shfl_down16(c);
        acc = over4(acc, over4(c, odd));
      }
      if (staged) __syncwarp();  // the box is overwritten by the next chunk
    }
    const uint32_t stations = parity ? 0u : (uint32_t)n;
    warp_stations += stations;
    if (parity || !in_img) continue;
    const long long pix = (long long)py * a.camera.width + px;
    reinterpret_cast<float4*>(a.out_rgba)[pix] = acc;
  }
  if (a.out_station_total) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) warp_stations += __shfl_xor_sync(0xffffffffu, warp_stations, off);
    if (lane == 0 && warp_stations) atomicAdd(a.out_station_total, warp_stations);
  }
}

template <int LINE>
static int launch_staged_l(const isc_render_args* a, const FastField& F, cudaStream_t st) {
  const int tw_log2 = 3;
  const int tw = 1 << tw_log2, th = 16 >> tw_log2;
  int tiles_x = (a->camera.width + tw - 1) / tw, tiles_y = (a->camera.height + th - 1) / th;
  int tile_x0 = 0, tile_y0 = 0;
  int rx0, ry0, rx1, ry1;
  if (brick_screen_rect(a, rx0, ry0, rx1, ry1)) {
    ISC_CUDA_CHECK(cudaMemsetAsync(a->out_rgba, 0, (size_t)a->camera.width * a->camera.height * sizeof(float4), st));
    if (rx1 <= rx0 || ry1 <= ry0) return ISC_OK;
    tile_x0 = rx0 / tw;
    tile_y0 = ry0 / th;
    tiles_x = (rx1 + tw - 1) / tw - tile_x0;
    tiles_y = (ry1 + th - 1) / th - tile_y0;
  }
  const int super_x = (tiles_x + 7) / 8, super_y = (tiles_y + 7) / 8;
  const int n_codes = super_x * super_y * 64;
  const size_t smem = (LINE == 0 ? ISC_LUT_ENTRIES * sizeof(float4) : 0) +
                      (size_t)kStageWarps * ISC_STAGE_WARP_FLOATS * sizeof(float);
  ISC_CUDA_CHECK(cudaFuncSetAttribute(march_staged_kernel<LINE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
  int dev = 0, sms = 148, per_sm = 1;
  ISC_CUDA_CHECK(cudaGetDevice(&dev));
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, march_staged_kernel<LINE>, kStageThreads, smem);
  int grid = sms * (per_sm > 0 ? per_sm : 1);
  const int need = (n_codes + kStageWarps - 1) / kStageWarps;
  if (grid > need) grid = need > 0 ? need : 1;
  march_staged_kernel<LINE><<<grid, kStageThreads, smem, st>>>(*a, F, tiles_x, tiles_y, super_x, n_codes, tw_log2,
                                                               tile_x0, tile_y0);
  ISC_CUDA_CHECK(cudaGetLastError());
  return ISC_OK;
}

// f32 scalar, guarded trilinear, no early termination; `lines` as in
// march.cu launch_line (0 = shared-memory LUT).
int launch_staged(int lines, const isc_render_args* a, const FastField& F, cudaStream_t st) {
  switch (lines) {
    case 1: return launch_staged_l<1>(a, F, st);
    case 2: return launch_staged_l<2>(a, F, st);
    case 3: return launch_staged_l<3>(a, F, st);
    case 4: return launch_staged_l<4>(a, F, st);
    default: return launch_staged_l<0>(a, F, st);
  }
}

}  // namespace isc
