// b8_probe.cu -- measures (on the GPU) which shared-memory byte each lane /
// register byte receives from the sm_100a 8-bit ldmatrix / stmatrix forms,
// the tiles the register-faithful path would left-divide by (DESIGN 8b:
// ".b8 tiles").  The PTX manual is not available offline, so the mapping is
// read off the hardware: smem byte i holds i (i < 256); for stores each lane
// writes bytes (lane << 2 | byte).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -o b8_probe b8_probe.cu
#include <cstdint>
#include <cstdio>

__global__ void ld_m16n16_trans(uint32_t* out) {
  __shared__ __align__(128) uint8_t sm[256];
  for (int i = threadIdx.x; i < 256; i += 32) sm[i] = (uint8_t)i;
  __syncwarp();
  const int lane = threadIdx.x;
  uint32_t addr = (uint32_t)__cvta_generic_to_shared(sm) + (lane & 15) * 16;
  uint32_t r0, r1;
  asm volatile("ldmatrix.sync.aligned.m16n16.x1.trans.shared.b8 {%0,%1}, [%2];"
               : "=r"(r0), "=r"(r1) : "r"(addr));
  out[lane * 2] = r0;
  out[lane * 2 + 1] = r1;
}

__global__ void st_m16n8_trans(uint32_t* out) {
  __shared__ __align__(128) uint8_t sm[256];
  for (int i = threadIdx.x; i < 256; i += 32) sm[i] = 0xff;
  __syncwarp();
  const int lane = threadIdx.x;
  // row addresses 16 B apart (8-byte spacing faults: misaligned address)
  uint32_t addr = (uint32_t)__cvta_generic_to_shared(sm) + (lane & 15) * 16;
  uint32_t v = 0;
  for (int b = 0; b < 4; ++b) v |= (uint32_t)((lane << 2) | b) << (8 * b);
  asm volatile("stmatrix.sync.aligned.m16n8.x1.trans.shared.b8 [%0], {%1};" ::"r"(addr), "r"(v) : "memory");
  __syncwarp();
  for (int i = lane; i < 256; i += 32) out[i] = sm[i];
}

int main() {
  uint32_t* d;
  uint32_t h[256];
  cudaMalloc(&d, 1024);
  cudaMemset(d, 0, 1024);
  ld_m16n16_trans<<<1, 32>>>(d);
  cudaMemcpy(h, d, 256, cudaMemcpyDeviceToHost);
  printf("{\"ldmatrix.m16n16.x1.trans.b8\": [");
  for (int l = 0; l < 32; ++l) {
    printf("%s[", l ? "," : "");
    for (int b = 0; b < 8; ++b) printf("%s%u", b ? "," : "", (h[l * 2 + b / 4] >> (8 * (b % 4))) & 255);
    printf("]");
  }
  printf("],\n");
  st_m16n8_trans<<<1, 32>>>(d);
  cudaMemcpy(h, d, 1024, cudaMemcpyDeviceToHost);
  printf(" \"stmatrix.m16n8.x1.trans.b8\": [");
  for (int i = 0; i < 256; ++i) printf("%s%u", i ? "," : "", h[i]);
  printf("],\n \"error\": \"%s\"}\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
