// bankprobe.cu -- shared-memory bank-model micro-benchmark (diagnostic tool,
// not part of libll_b200).  Each warp of the block executes `n_instr`
// ld.shared / st.shared instructions of width W bytes whose per-lane byte
// offsets come from `offs` ([warps][n_instr][32]); ncu's wavefront counters
// on this kernel give the hardware's cost of exactly those address patterns.
#include <cuda_runtime.h>
#include <cstdint>

template <int W, bool STORE>
__global__ void probe(const uint32_t* __restrict__ offs, int n_instr, int reps, uint32_t* out) {
  extern __shared__ __align__(16) uint8_t sm[];
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = i * 2654435761u;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t o[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) o[i] = i < n_instr ? offs[(warp * n_instr + i) * 32 + lane] : 0;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm);
  uint32_t acc = 0;
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      if (i >= n_instr) break;
      const uint32_t a = base + o[i];
      if (STORE) {
        if (W == 16) asm volatile("st.shared.v4.b32 [%0], {%1,%1,%1,%1};" ::"r"(a), "r"(acc + r) : "memory");
        else if (W == 8) asm volatile("st.shared.v2.b32 [%0], {%1,%1};" ::"r"(a), "r"(acc + r) : "memory");
        else asm volatile("st.shared.b32 [%0], %1;" ::"r"(a), "r"(acc + r) : "memory");
      } else {
        uint32_t x, y, z, w;
        if (W == 16) {
          asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(x), "=r"(y), "=r"(z), "=r"(w) : "r"(a));
          acc ^= x ^ y ^ z ^ w;
        } else if (W == 8) {
          asm volatile("ld.shared.v2.b32 {%0,%1}, [%2];" : "=r"(x), "=r"(y) : "r"(a));
          acc ^= x ^ y;
        } else {
          asm volatile("ld.shared.b32 %0, [%1];" : "=r"(x) : "r"(a));
          acc ^= x;
        }
      }
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

extern "C" int bankprobe(int width, int store, const uint32_t* offs_dev, int warps, int n_instr,
                         int reps, int blocks, uint32_t* out_dev) {
  const size_t sm = 65536;
  dim3 g(blocks), b(32 * warps);
#define L(WW, SS)                                                                         \
  do {                                                                                     \
    cudaFuncSetAttribute(probe<WW, SS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
    probe<WW, SS><<<g, b, sm>>>(offs_dev, n_instr, reps, out_dev);                       \
  } while (0)
  if (width == 16) { if (store) L(16, true); else L(16, false); }
  else if (width == 8) { if (store) L(8, true); else L(8, false); }
  else { if (store) L(4, true); else L(4, false); }
#undef L
  return (int)cudaDeviceSynchronize();
}
