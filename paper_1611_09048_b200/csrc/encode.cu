// Frame quantisation for the encode step that follows compositing on rank 0:
// to_rgba8 = round(clip(rgba, 0, 1) * 255) with numpy's round-half-to-even
// (runtime.py:66-67).  One float4 -> uchar4 per thread; the 8-bit frame is a
// quarter of the float frame, which is what crosses PCIe to the encoder.
#include "common.cuh"

namespace isc {

__device__ __forceinline__ unsigned char q8(float v) {
  v = fminf(fmaxf(v, 0.0f), 1.0f) * 255.0f;
  return (unsigned char)__float2int_rn(v);   // round half to even
}

__global__ void to_rgba8_kernel(const float4* __restrict__ in, uchar4* __restrict__ out, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const float4 c = __ldcs(in + i);
    out[i] = make_uchar4(q8(c.x), q8(c.y), q8(c.z), q8(c.w));
  }
}

}  // namespace isc

using namespace isc;

extern "C" int isc_to_rgba8(const float* rgba, uint8_t* out, int64_t n_pixels, void* stream) {
  if (n_pixels < 0 || (n_pixels > 0 && (!rgba || !out))) return fail(ISC_E_VALUE, "bad to_rgba8 arguments");
  if (n_pixels == 0) return ISC_OK;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  long long grid = (n_pixels + 255) / 256;
  if (grid > sms * 16LL) grid = sms * 16LL;
  to_rgba8_kernel<<<(int)grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const float4*>(rgba), reinterpret_cast<uchar4*>(out), n_pixels);
  ISC_CUDA_CHECK(cudaGetLastError());
  return ISC_OK;
}
