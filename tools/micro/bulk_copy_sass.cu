// Per-lane 1-D bulk copies (cp.async.bulk, the only TMA form a 4104-byte row pitch allows):
// compile with nvcc -gencode arch=compute_100a,code=sm_100a -cubin and read the SASS -- each
// lane's copy becomes one iteration of an ELECT / R2UR.BROADCAST x3 / UBLKCP / BRA.U.ANY loop
// (UBLKCP takes uniform operands), i.e. the copies of a warp serialise.
#include <cstdint>
__global__ void k(const float* __restrict__ g, float* out, int pitch) {
  extern __shared__ __align__(16) float box[];
  __shared__ __align__(8) unsigned long long mbar;
  const int lane = threadIdx.x & 31;
  const unsigned mb = (unsigned)__cvta_generic_to_shared(&mbar);
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(mb));
  __syncthreads();
  if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(mb), "r"(32 * 64));
  __syncwarp();
  const float* src = g + (size_t)lane * pitch;
  const unsigned dst = (unsigned)__cvta_generic_to_shared(box + lane * 16);
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 64, [%2];"
               ::"r"(dst), "l"(src), "r"(mb) : "memory");
  asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared.b64 p, [%0], 0;\n @!p bra W;\n}" ::"r"(mb));
  out[threadIdx.x] = box[threadIdx.x * 3 % 512];
}
