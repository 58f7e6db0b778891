// bwprobe.cu -- HBM ceilings for the traffic mixes of the hot path
// (standalone; nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o bwprobe bwprobe.cu).
//
//   copy       1 : 1 read : write, 16 B per thread per access
//   write      write only
//   r1w4_coal  read 16 B, write 64 B per thread; each warp store instruction
//              covers 512 contiguous bytes (fully coalesced)
//   r1w4_lane  read 16 B, write 64 B per thread as 4 x 16 B at +0/16/32/48 of
//              the thread's own 64 B
//   r1w4_pair  lane pairs fill one 32-byte sector per store instruction (the
//              upcast kernel's store pattern)
//   r1w4_quad  lane quads fill 64 contiguous bytes per store instruction
//   copy256    1 : 1 with sm_100 256-bit loads and stores (32 B per thread)
//   r1w4_v8    read 16 B, write the thread's own 64 B as two 256-bit stores
//              (the upcast kernel's store pattern since LL_UP_V8)
// Prints one JSON line per case: GB/s = (read + write bytes) / time, best of
// 20 launches over two rotating buffer sets larger than L2.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ void stg(uint4* p, uint4 v) {
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};"
               :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

__global__ void k_copy(const uint4* __restrict__ a, uint4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    stg(b + i, ldg_stream(a + i));
}
__global__ void k_write(uint4* __restrict__ b, size_t n, uint32_t v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    stg(b + i, make_uint4(v, v + 1, v + 2, v + 3));
}
// n = number of 16-byte source vectors
__global__ void k_r1w4_coal(const uint4* __restrict__ a, uint4* __restrict__ b, size_t n) {
  const int lane = threadIdx.x & 31;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 x = ldg_stream(a + i);
    const size_t w0 = (i - lane) * 4;  // the warp's 32 x 64 B output block
#pragma unroll
    for (int q = 0; q < 4; ++q)
      stg(b + w0 + q * 32 + lane, make_uint4(x.x ^ q, x.y, x.z, x.w));
  }
}
__global__ void k_r1w4_lane(const uint4* __restrict__ a, uint4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 x = ldg_stream(a + i);
#pragma unroll
    for (int q = 0; q < 4; ++q) stg(b + 4 * i + q, make_uint4(x.x ^ q, x.y, x.z, x.w));
  }
}

// lane pairs: instruction q writes one whole 32-byte sector per pair (the
// upcast kernel's pattern): lane 2i+o stores 16 B at 64*(2i + (q>>1)) + 32*(q&1) + 16*o
__global__ void k_r1w4_pair(const uint4* __restrict__ a, uint4* __restrict__ b, size_t n) {
  const int o = threadIdx.x & 1;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 x = ldg_stream(a + i);
    const size_t pair0 = (i - o) * 4;  // the pair's 2 x 64 B block, in 16-B units
#pragma unroll
    for (int q = 0; q < 4; ++q)
      stg(b + pair0 + 4 * (q >> 1) + 2 * (q & 1) + o, make_uint4(x.x ^ q, x.y, x.z, x.w));
  }
}
// quads: instruction q writes 64 contiguous bytes per 4 lanes
__global__ void k_r1w4_quad(const uint4* __restrict__ a, uint4* __restrict__ b, size_t n) {
  const int o = threadIdx.x & 3;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 x = ldg_stream(a + i);
    const size_t q0 = (i - o) * 4;
#pragma unroll
    for (int q = 0; q < 4; ++q) stg(b + q0 + 4 * q + o, make_uint4(x.x ^ q, x.y, x.z, x.w));
  }
}

struct alignas(32) u8x32 { uint32_t w[8]; };
__device__ __forceinline__ u8x32 ldg256(const u8x32* p) {
  u8x32 v;
  asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v.w[0]), "=r"(v.w[1]), "=r"(v.w[2]), "=r"(v.w[3]), "=r"(v.w[4]), "=r"(v.w[5]),
                 "=r"(v.w[6]), "=r"(v.w[7]) : "l"(p));
  return v;
}
__device__ __forceinline__ void stg256(u8x32* p, const u8x32& v) {
  asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
               :: "l"(p), "r"(v.w[0]), "r"(v.w[1]), "r"(v.w[2]), "r"(v.w[3]), "r"(v.w[4]), "r"(v.w[5]),
                  "r"(v.w[6]), "r"(v.w[7]) : "memory");
}
__global__ void k_copy256(const u8x32* __restrict__ a, u8x32* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    stg256(b + i, ldg256(a + i));
}
__global__ void k_r1w4_v8(const uint4* __restrict__ a, u8x32* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 x = ldg_stream(a + i);
    u8x32 v{{x.x, x.y, x.z, x.w, x.x ^ 1, x.y, x.z, x.w}};
    stg256(b + 2 * i, v);
    v.w[0] ^= 2;
    stg256(b + 2 * i + 1, v);
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t in_bytes = (size_t)512 << 20, out_bytes = 4 * in_bytes;
  uint4 *a[2], *b[2];
  for (int s = 0; s < 2; ++s) {
    cudaMalloc(&a[s], out_bytes);
    cudaMalloc(&b[s], out_bytes);
    cudaMemset(a[s], 1, out_bytes);
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int threads = 256;
  for (int bps : {4, 8, 16}) {
    const int grid = sms * bps;
    auto run = [&](const char* name, double bytes, auto launch) {
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
      printf("{\"case\": \"%s\", \"blocks_per_sm\": %d, \"ms\": %.4f, \"GBps\": %.1f}\n", name, bps, best,
             bytes / best / 1e6);
    };
    const size_t nv = in_bytes / 16;
    run("copy 2GiB+2GiB", 2.0 * out_bytes, [&](int s) { k_copy<<<grid, threads>>>(a[s], b[s], out_bytes / 16); });
    run("write 2GiB", 1.0 * out_bytes, [&](int s) { k_write<<<grid, threads>>>(b[s], out_bytes / 16, s); });
    run("r1w4_coal 512MiB->2GiB", 5.0 * in_bytes, [&](int s) { k_r1w4_coal<<<grid, threads>>>(a[s], b[s], nv); });
    run("r1w4_lane 512MiB->2GiB", 5.0 * in_bytes, [&](int s) { k_r1w4_lane<<<grid, threads>>>(a[s], b[s], nv); });
    run("r1w4_pair 512MiB->2GiB", 5.0 * in_bytes, [&](int s) { k_r1w4_pair<<<grid, threads>>>(a[s], b[s], nv); });
    run("r1w4_quad 512MiB->2GiB", 5.0 * in_bytes, [&](int s) { k_r1w4_quad<<<grid, threads>>>(a[s], b[s], nv); });
    run("copy256 2GiB+2GiB", 2.0 * out_bytes, [&](int s) { k_copy256<<<grid, threads>>>((const u8x32*)a[s], (u8x32*)b[s], out_bytes / 32); });
    run("r1w4_v8 512MiB->2GiB", 5.0 * in_bytes, [&](int s) { k_r1w4_v8<<<grid, threads>>>(a[s], (u8x32*)b[s], nv); });
  }
  cudaError_t err = cudaDeviceSynchronize();
  if (err != cudaSuccess) {
    printf("{\"error\": \"%s\"}\n", cudaGetErrorString(err));
    return 1;
  }
  return 0;
}
