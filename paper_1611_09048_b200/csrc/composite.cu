// K5-K7: sort-last compositing over peer memory.
//
//   isc_over            over_arrays           compositing.py:31-33
//   isc_composite_fold  composite_sequential  compositing.py:66-77
//   isc_binary_swap     binary_swap           compositing.py:107-181
//   isc_direct_send     _direct_send          compositing.py:184-194
//
// The swap is ONE persistent kernel per rank: every round pulls the
// partner's half-span straight out of the partner's image through its
// peer-mapped pointer (NVLink 5 loads on a multi-GPU box), composites it with
// the local half in visibility order and writes the result in place, so the
// transfer and the `over` are the same instruction stream.  After the last
// round each rank stores its final span directly into rank 0's output (the
// collection step of compositing.py:169-181).
//
// Slices.  The image is cut into n_ctas contiguous slices and CTA b of every
// rank runs the reference's binary swap on slice b alone: round r halves the
// slice-b span at (lo+hi)/2 and keeps the high half iff bit r of the rank's
// visibility position is set, exactly as compositing.py:145-160 does on the
// whole image.  Every pixel therefore sees the same tree of `over`s as the
// reference (bit-identical results); only which rank holds which pixels at
// the end differs, and rank 0's output is the same full frame.  CTA b only
// ever reads and writes slice b, so the ordering is per slice: CTA b
// publishes "slice b reached stage s" with a system-scope release add on its
// own counter, and reads a peer's slice b after an acquire load of that
// peer's slice-b counter.  There is no grid-wide barrier inside a rank, so
// nothing requires the grid to be co-resident: with CTAs dispatched in index
// order the lowest unfinished slice always runs on every rank, which keeps a
// swap that shares the GPU with other kernels (in situ: the simulation's)
// progressing.  Spin-waits are bounded by a timeout that surfaces as
// TransportError instead of a hung GPU.
#include <cstring>

#include "common.cuh"

namespace isc {

// Flag block of one rank: kCtrlWords control words (kErrWord = transport
// error), then per-slice arrival counters, word kCtrlWords + stage *
// ISC_MAX_SWAP_CTAS + slice.  Stages: 0 image ready, r+1 round r done,
// rounds+1 final span stored into rank 0's output, kRootReadStage rank 0 has
// read the slice (direct send).  Every counter grows by exactly one per
// epoch, so "stage reached in epoch e" is "counter >= e".
constexpr int kCtrlWords = 16;
constexpr int kErrWord = 9;
constexpr int kEpochWord = 10;  // device-resident epoch (isc_swap_epoch_bump)
constexpr int kStages = ISC_SWAP_STAGES;
constexpr int kRootReadStage = kStages - 1;
constexpr int kFlagWords = kCtrlWords + kStages * ISC_MAX_SWAP_CTAS;
static_assert(ISC_MAX_ROUNDS + 2 <= kRootReadStage, "stage words overlap");

__device__ __forceinline__ unsigned long long* stage_word(unsigned long long* flags, int stage, int slice) {
  return flags + kCtrlWords + stage * ISC_MAX_SWAP_CTAS + slice;
}

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Thread 0 spins until *p >= target; returns false on timeout (and records
// the error in the local flag block).  Caller must __syncthreads afterwards.
__device__ bool wait_at_least(const unsigned long long* p, unsigned long long target, long long timeout_ns,
                              unsigned long long* my_flags) {
  const unsigned long long t0 = global_ns();
  unsigned int backoff = 32;
  while (ld_acquire_sys(p) < target) {
    if ((long long)(global_ns() - t0) > timeout_ns) {
      atomicExch(my_flags + kErrWord, 1ull);
      return false;
    }
    __nanosleep(backoff);
    if (backoff < 1024) backoff <<= 1;
  }
  return true;
}

// Whole CTA: every thread's prior writes, then thread 0 bumps the counter.
__device__ __forceinline__ void publish(unsigned long long* counter) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    red_release_sys(counter, 1ull);
  }
}

// Returns false if any thread of the CTA saw a timeout.
__device__ __forceinline__ bool cta_wait(const unsigned long long* p, unsigned long long target, long long tmo,
                                         unsigned long long* my_flags) {
  __shared__ int ok;
  if (threadIdx.x == 0) ok = wait_at_least(p, target, tmo, my_flags) ? 1 : 0;
  __syncthreads();
  const bool r = ok != 0;
  __syncthreads();
  return r;
}

__global__ void over_kernel(float4* dst, const float4* front, const float4* back, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    dst[i] = over4(__ldcg(front + i), __ldcg(back + i));
}

struct FoldArgs {
  const float4* img[ISC_MAX_RANKS];
  int n;
};

__global__ void fold_kernel(float4* out, const __grid_constant__ FoldArgs f, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int r = 0; r < f.n; ++r) acc = over4(acc, __ldcg(f.img[r] + i));
    out[i] = acc;
  }
}

// out[i] = front/back over of mine[i] and theirs[i] for i in [c0, c1): 4
// pixels (8 independent 16-byte loads) per thread in flight.
__device__ __forceinline__ void over_span(float4* mine, const float4* theirs, long long c0, long long c1,
                                          bool partner_front) {
  const long long stride = blockDim.x;
  long long i = c0 + threadIdx.x;
  for (; i + 3 * stride < c1; i += 4 * stride) {
    float4 m[4], t[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      m[u] = __ldcg(mine + i + u * stride);
      t[u] = __ldcg(theirs + i + u * stride);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) mine[i + u * stride] = partner_front ? over4(t[u], m[u]) : over4(m[u], t[u]);
  }
  for (; i < c1; i += stride) {
    const float4 m = __ldcg(mine + i), t = __ldcg(theirs + i);
    mine[i] = partner_front ? over4(t, m) : over4(m, t);
  }
}

__device__ __forceinline__ void copy_span(float4* out, const float4* in, long long c0, long long c1) {
  const long long stride = blockDim.x;
  long long i = c0 + threadIdx.x;
  for (; i + 3 * stride < c1; i += 4 * stride) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = __ldcg(in + i + u * stride);
#pragma unroll
    for (int u = 0; u < 4; ++u) out[i + u * stride] = v[u];
  }
  for (; i < c1; i += stride) out[i] = __ldcg(in + i);
}

// Slice b of n pixels cut into `parts` contiguous slices.
__device__ __forceinline__ void slice_of(long long n, int parts, int b, long long& a, long long& e) {
  const long long per = (n + parts - 1) / parts;
  a = min(n, per * b);
  e = min(n, a + per);
}

__global__ void __launch_bounds__(512) swap_kernel(const __grid_constant__ isc_swap_args a) {
  const int R = a.size;
  const int b = blockIdx.x;
  int v = 0;
  for (int i = 0; i < R; ++i)
    if (a.order[i] == a.rank) v = i;
  int rounds = 0;
  while ((1 << rounds) < R) ++rounds;
  unsigned long long* me = a.flags[a.rank];
  const unsigned long long target = a.epoch ? (unsigned long long)a.epoch : __ldcg(me + kEpochWord);
  float4* mine = reinterpret_cast<float4*>(a.image[a.rank]);

  // slice b of the image is ready (stream-ordered after the render)
  if (a.publish_ready) publish(stage_word(me, 0, b));

  long long lo, hi;
  slice_of(a.n_pixels, a.n_ctas, b, lo, hi);
  for (int r = 0; r < rounds; ++r) {
    const int bit = 1 << r;
    const int pv = v ^ bit;
    const long long mid = (lo + hi) / 2;          // compositing.py:150
    const bool keep_high = (v & bit) != 0;
    const long long klo = keep_high ? mid : lo, khi = keep_high ? hi : mid;
    if (r >= a.round_begin && r < a.round_end) {
      const int partner = a.order[pv];
      // the partner finished round r-1 on slice b (r = 0: its image is
      // ready); this CTA's own round r-1 precedes it in program order (or,
      // launched round by round, in stream order)
      if (!cta_wait(stage_word(a.flags[partner], r, b), target, a.timeout_ns, me)) return;
      over_span(mine, reinterpret_cast<const float4*>(a.image[partner]), klo, khi, pv < v);
      publish(stage_word(me, r + 1, b));
    }
    lo = klo;
    hi = khi;
  }

  if (a.collect) {
    copy_span(reinterpret_cast<float4*>(a.root_out), mine, lo, hi);
    publish(stage_word(me, rounds + 1, b));
  }

  if (a.finish) {
    if (a.rank == 0) {
      // every rank's final span of slice b has landed in the output
      for (int q = 0; q < R; ++q)
        if (!cta_wait(stage_word(a.flags[q], rounds + 1, b), target, a.timeout_ns, me)) return;
    } else {
      // every partner has finished reading this rank's slice b
      for (int r = 0; r < rounds; ++r)
        if (!cta_wait(stage_word(a.flags[a.order[v ^ (1 << r)]], r + 1, b), target, a.timeout_ns, me)) return;
    }
  }
}

__global__ void __launch_bounds__(512) direct_send_kernel(const __grid_constant__ isc_swap_args a) {
  const int b = blockIdx.x;
  unsigned long long* me = a.flags[a.rank];
  const unsigned long long target = a.epoch ? (unsigned long long)a.epoch : __ldcg(me + kEpochWord);
  if (a.publish_ready) publish(stage_word(me, 0, b));
  long long c0, c1;
  slice_of(a.n_pixels, a.n_ctas, b, c0, c1);
  if (a.rank == 0) {
    for (int q = 0; q < a.size; ++q)
      if (!cta_wait(stage_word(a.flags[q], 0, b), target, a.timeout_ns, me)) return;
    float4* out = reinterpret_cast<float4*>(a.root_out);
    for (long long i = c0 + threadIdx.x; i < c1; i += blockDim.x) {
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int r = 0; r < a.size; ++r)
        acc = over4(acc, __ldcg(reinterpret_cast<const float4*>(a.image[a.order[r]]) + i));
      out[i] = acc;
    }
    publish(stage_word(me, kRootReadStage, b));
  } else if (a.finish) {
    cta_wait(stage_word(a.flags[0], kRootReadStage, b), target, a.timeout_ns, me);
  }
}

static int grid_for(long long n) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  long long g = (n + 255) / 256;
  const long long cap = (long long)sms * 8;
  return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

static int check_swap(const isc_swap_args* a, bool pow2) {
  if (!a) return fail(ISC_E_VALUE, "null swap args");
  if (a->size < 1 || a->size > ISC_MAX_RANKS) return fail(ISC_E_COMPOSITE, "world size out of range");
  if (a->rank < 0 || a->rank >= a->size) return fail(ISC_E_COMPOSITE, "rank out of range");
  if (pow2 && (a->size & (a->size - 1))) return fail(ISC_E_COMPOSITE, "binary swap needs a power-of-two size");
  if (a->n_ctas < 1 || a->n_ctas > ISC_MAX_SWAP_CTAS) return fail(ISC_E_COMPOSITE, "n_ctas out of range");
  if (a->epoch < 0) return fail(ISC_E_COMPOSITE, "epoch must be >= 1 (or 0: device-resident)");
  unsigned seen = 0;
  unsigned long long seen_hi = 0;
  for (int i = 0; i < a->size; ++i) {
    const int o = a->order[i];
    if (o < 0 || o >= a->size) return fail(ISC_E_COMPOSITE, "order entry out of range");
    if (o < 32) { if (seen & (1u << o)) return fail(ISC_E_COMPOSITE, "order is not a permutation"); seen |= 1u << o; }
    else { if (seen_hi & (1ull << (o - 32))) return fail(ISC_E_COMPOSITE, "order is not a permutation"); seen_hi |= 1ull << (o - 32); }
    if (!a->image[i] || !a->flags[i]) return fail(ISC_E_COMPOSITE, "missing image/flag pointer");
  }
  return ISC_OK;
}

}  // namespace isc

using namespace isc;

extern "C" int isc_over(float* dst, const float* front, const float* back, int64_t n, void* stream) {
  if (n < 0 || (n > 0 && (!dst || !front || !back))) return fail(ISC_E_VALUE, "bad over arguments");
  if (n == 0) return ISC_OK;
  over_kernel<<<grid_for(n), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<float4*>(dst), reinterpret_cast<const float4*>(front), reinterpret_cast<const float4*>(back), n);
  ISC_CUDA_CHECK(cudaGetLastError());
  return ISC_OK;
}

extern "C" int isc_composite_fold(float* out, const float* const* images, int32_t n_images, int64_t n, void* stream) {
  if (!out || !images || n_images < 1 || n_images > ISC_MAX_RANKS || n < 0)
    return fail(ISC_E_COMPOSITE, "bad fold arguments");
  if (n == 0) return ISC_OK;
  FoldArgs f;
  f.n = n_images;
  for (int i = 0; i < n_images; ++i) {
    if (!images[i]) return fail(ISC_E_COMPOSITE, "null image pointer");
    f.img[i] = reinterpret_cast<const float4*>(images[i]);
  }
  fold_kernel<<<grid_for(n), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(reinterpret_cast<float4*>(out), f, n);
  ISC_CUDA_CHECK(cudaGetLastError());
  return ISC_OK;
}

extern "C" int isc_binary_swap(const isc_swap_args* a, void* stream) {
  int st = check_swap(a, true);
  if (st != ISC_OK) return st;
  if (a->collect && !a->root_out) return fail(ISC_E_COMPOSITE, "collect needs root_out");
  swap_kernel<<<a->n_ctas, 512, 0, reinterpret_cast<cudaStream_t>(stream)>>>(*a);
  ISC_CUDA_CHECK(cudaGetLastError());
  return ISC_OK;
}

extern "C" int isc_direct_send(const isc_swap_args* a, void* stream) {
  int st = check_swap(a, false);
  if (st != ISC_OK) return st;
  if (a->rank == 0 && !a->root_out) return fail(ISC_E_COMPOSITE, "root needs root_out");
  direct_send_kernel<<<a->n_ctas, 512, 0, reinterpret_cast<cudaStream_t>(stream)>>>(*a);
  ISC_CUDA_CHECK(cudaGetLastError());
  return ISC_OK;
}

extern "C" int isc_flag_words(void) { return kFlagWords; }

extern "C" int isc_swap_status(unsigned long long* flags, void* stream, unsigned long long* pinned,
                               int32_t* out_code) {
  if (!flags || !out_code || !pinned) return fail(ISC_E_VALUE, "null argument");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  // pinned destination: a stream-ordered copy that never waits on other streams
  ISC_CUDA_CHECK(cudaMemcpyAsync(pinned, flags + kErrWord, sizeof(*pinned), cudaMemcpyDeviceToHost, s));
  ISC_CUDA_CHECK(cudaStreamSynchronize(s));
  const unsigned long long v = *pinned;
  *out_code = (int32_t)v;
  if (v) {
    ISC_CUDA_CHECK(cudaMemsetAsync(flags + kErrWord, 0, sizeof(unsigned long long), s));
    ISC_CUDA_CHECK(cudaStreamSynchronize(s));
  }
  return ISC_OK;
}

extern "C" int isc_swap_error_async(unsigned long long* flags, unsigned long long* pinned, void* stream) {
  if (!flags || !pinned) return fail(ISC_E_VALUE, "null argument");
  ISC_CUDA_CHECK(cudaMemcpyAsync(pinned, flags + kErrWord, sizeof(*pinned), cudaMemcpyDeviceToHost,
                                 reinterpret_cast<cudaStream_t>(stream)));
  return ISC_OK;
}

extern "C" int isc_swap_reset(unsigned long long* flags, void* stream) {
  if (!flags) return fail(ISC_E_VALUE, "null flag block");
  ISC_CUDA_CHECK(cudaMemsetAsync(flags, 0, sizeof(unsigned long long) * kFlagWords,
                                 reinterpret_cast<cudaStream_t>(stream)));
  return ISC_OK;
}

__global__ void epoch_bump_kernel(unsigned long long* flags) { flags[kEpochWord] += 1ull; }

extern "C" int isc_swap_epoch_bump(unsigned long long* flags, void* stream) {
  if (!flags) return fail(ISC_E_VALUE, "null flag block");
  epoch_bump_kernel<<<1, 1, 0, reinterpret_cast<cudaStream_t>(stream)>>>(flags);
  ISC_CUDA_CHECK(cudaGetLastError());
  return ISC_OK;
}

__global__ void occupy_kernel(long long ns) {
  const unsigned long long t0 = global_ns();
  while ((long long)(global_ns() - t0) < ns) __nanosleep(1000);
}

extern "C" int isc_debug_occupy(int32_t n_ctas, int32_t threads, int64_t ns, void* stream) {
  if (n_ctas < 1 || threads < 1 || threads > 1024 || ns < 0) return fail(ISC_E_VALUE, "bad occupy arguments");
  occupy_kernel<<<n_ctas, threads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(ns);
  ISC_CUDA_CHECK(cudaGetLastError());
  return ISC_OK;
}

extern "C" int isc_arena_alloc(size_t bytes, void** out_ptr) {
  if (!out_ptr || bytes == 0) return fail(ISC_E_VALUE, "bad arena request");
  ISC_CUDA_CHECK(cudaMalloc(out_ptr, bytes));
  ISC_CUDA_CHECK(cudaMemset(*out_ptr, 0, bytes));
  ISC_CUDA_CHECK(cudaDeviceSynchronize());
  return ISC_OK;
}

extern "C" int isc_arena_free(void* ptr) {
  if (ptr) ISC_CUDA_CHECK(cudaFree(ptr));
  return ISC_OK;
}

extern "C" int isc_ipc_handle(void* dev_ptr, unsigned char out[ISC_IPC_HANDLE_BYTES]) {
  static_assert(sizeof(cudaIpcMemHandle_t) == ISC_IPC_HANDLE_BYTES, "ipc handle size");
  if (!dev_ptr || !out) return fail(ISC_E_VALUE, "null argument");
  cudaIpcMemHandle_t h;
  ISC_CUDA_CHECK(cudaIpcGetMemHandle(&h, dev_ptr));
  memcpy(out, &h, sizeof(h));
  return ISC_OK;
}

extern "C" int isc_ipc_open(const unsigned char handle[ISC_IPC_HANDLE_BYTES], void** out_ptr) {
  if (!handle || !out_ptr) return fail(ISC_E_VALUE, "null argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  ISC_CUDA_CHECK(cudaIpcOpenMemHandle(out_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return ISC_OK;
}

extern "C" int isc_ipc_close(void* p) {
  if (p) ISC_CUDA_CHECK(cudaIpcCloseMemHandle(p));
  return ISC_OK;
}

extern "C" int isc_enable_peer_access(int peer) {
  cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return ISC_OK;
  }
  if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceEnablePeerAccess");
  return ISC_OK;
}
