// transpose_probe.cu -- ceilings for config 3's DRAM access pattern
// (standalone; nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o transpose_probe transpose_probe.cu)
//
// 8192 x 8192 2-byte elements, tiles of T x T (T = 64 or 128), one tile per
// 256-thread CTA (grid = all tiles), staged through a padded shared-memory
// tile.  Cases:
//   tiled_copy   tile rows -> the same tile rows (the transpose's DRAM pattern
//                on both sides, no transposition): 2*T-byte row segments
//   transpose    tile rows -> tile columns (row-major -> column-major)
//   *_v8         the same with 256-bit (32-byte) global accesses
//   flat_copy    contiguous grid-stride copy, 16 B (reference)
// Prints one JSON line per case: GB/s = 2 * 128 MiB / time, best of 20, two
// rotating buffer sets (> L2).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 8192;

template <int T, bool TRANSPOSE, int VB>
__global__ void __launch_bounds__(256) k_tile(const uint16_t* __restrict__ a, uint16_t* __restrict__ b) {
  // VB = bytes per global access (16 or 32); EV elements per access
  constexpr int EV = VB / 2;
  constexpr int PER_ROW = T / EV;             // accesses per tile row
  constexpr int ITEMS = T * PER_ROW / 256;    // accesses per thread
  __shared__ uint16_t s[T][T + 8];
  const int tiles_per_row = N / T;
  const int ti = blockIdx.x / tiles_per_row, tj = blockIdx.x % tiles_per_row;
  const int t = threadIdx.x;
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const int idx = t + 256 * k;
    const int r = idx / PER_ROW, c = (idx % PER_ROW) * EV;
    const uint16_t* p = a + (size_t)(ti * T + r) * N + tj * T + c;
    if constexpr (VB == 16) {
      uint4 v;
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
      const uint16_t* e = reinterpret_cast<const uint16_t*>(&v);
#pragma unroll
      for (int q = 0; q < EV; ++q) s[r][c + q] = e[q];
    } else {
      uint32_t w[8];
      asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
                   : "l"(p));
      const uint16_t* e = reinterpret_cast<const uint16_t*>(w);
#pragma unroll
      for (int q = 0; q < EV; ++q) s[r][c + q] = e[q];
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const int idx = t + 256 * k;
    const int r = idx / PER_ROW, c = (idx % PER_ROW) * EV;
    uint16_t e[EV];
#pragma unroll
    for (int q = 0; q < EV; ++q) e[q] = TRANSPOSE ? s[c + q][r] : s[r][c + q];
    // destination: transpose writes column r of the source tile as row r of
    // the destination tile (tile (tj, ti)); the copy writes tile (ti, tj)
    uint16_t* p = TRANSPOSE ? b + (size_t)(tj * T + r) * N + ti * T + c
                            : b + (size_t)(ti * T + r) * N + tj * T + c;
    const uint32_t* w = reinterpret_cast<const uint32_t*>(e);
    if constexpr (VB == 16)
      asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(p), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]) : "memory");
    else
      asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" :: "l"(p), "r"(w[0]), "r"(w[1]), "r"(w[2]),
                   "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]) : "memory");
  }
}

__global__ void k_flat(const uint4* __restrict__ a, uint4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(a + i));
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(b + i), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t bytes = (size_t)N * N * 2;
  uint16_t *a[2], *b[2];
  for (int s = 0; s < 2; ++s) {
    cudaMalloc(&a[s], bytes);
    cudaMalloc(&b[s], bytes);
    cudaMemset(a[s], 1, bytes);
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, auto launch) {
    float best = 1e30f;
    for (int it = 0; it < 22; ++it) {
      cudaEventRecord(e0);
      launch(it & 1);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (it >= 2 && ms < best) best = ms;
    }
    printf("{\"case\": \"%s\", \"ms\": %.4f, \"GBps\": %.1f}\n", name, best, 2.0 * bytes / best / 1e6);
  };
  run("flat_copy 16B", [&](int s) { k_flat<<<sms * 16, 256>>>((const uint4*)a[s], (uint4*)b[s], bytes / 16); });
  run("tiled_copy T64 16B", [&](int s) { k_tile<64, false, 16><<<(N / 64) * (N / 64), 256>>>(a[s], b[s]); });
  run("transpose T64 16B", [&](int s) { k_tile<64, true, 16><<<(N / 64) * (N / 64), 256>>>(a[s], b[s]); });
  run("tiled_copy T128 16B", [&](int s) { k_tile<128, false, 16><<<(N / 128) * (N / 128), 256>>>(a[s], b[s]); });
  run("transpose T128 16B", [&](int s) { k_tile<128, true, 16><<<(N / 128) * (N / 128), 256>>>(a[s], b[s]); });
  run("tiled_copy T64 32B", [&](int s) { k_tile<64, false, 32><<<(N / 64) * (N / 64), 256>>>(a[s], b[s]); });
  run("transpose T64 32B", [&](int s) { k_tile<64, true, 32><<<(N / 64) * (N / 64), 256>>>(a[s], b[s]); });
  run("tiled_copy T128 32B", [&](int s) { k_tile<128, false, 32><<<(N / 128) * (N / 128), 256>>>(a[s], b[s]); });
  run("transpose T128 32B", [&](int s) { k_tile<128, true, 32><<<(N / 128) * (N / 128), 256>>>(a[s], b[s]); });
  cudaError_t err = cudaDeviceSynchronize();
  if (err != cudaSuccess) {
    printf("{\"error\": \"%s\"}\n", cudaGetErrorString(err));
    return 1;
  }
  return 0;
}
