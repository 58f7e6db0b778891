struct TileTab { long long src, dst, sc; };
struct TileMap { long long n_tiles; int n_bits; int n_tab; long long bss, bsd; TileTab tab[3][256]; };
extern "C" __global__ void __launch_bounds__(256) ll_shfl_hbm(
    const __grid_constant__ TileMap tm, const unsigned char* __restrict__ src,
    unsigned char* __restrict__ dst, long long n_groups, long long t0, long long t1,
    long long src_shift, long long dst_shift, long long pf_ctas) {
  const int lane = threadIdx.x & 31;
  const long long gid = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (gid >= n_groups) return;
  unsigned ld_off = 0, st_off = 0, fb = 0, fz = 0, fd = 0;
  if (lane & 1) { ld_off += 16u; st_off += 16u; fb ^= 1u; fz ^= 0u; fd ^= 4u; }
  if (lane & 2) { ld_off += 32u; st_off += 32u; fb ^= 2u; fz ^= 1u; fd ^= 1u; }
  if (lane & 4) { ld_off += 64u; st_off += 64u; fb ^= 0u; fz ^= 2u; fd ^= 2u; }
  if (lane & 8) { ld_off += 16384u; st_off += 128u; fb ^= 0u; fz ^= 0u; fd ^= 8u; }
  if (lane & 16) { ld_off += 32768u; st_off += 256u; fb ^= 0u; fz ^= 0u; fd ^= 16u; }
  const unsigned char* sthr = src + ld_off - src_shift;
  unsigned char* dthr = dst + st_off - dst_shift;
  const long long rmask = (1LL << tm.n_bits) - 1;
  { const long long t = t0 + gid; if (t < t1 && blockIdx.x < pf_ctas) {
    const long long inst = t >> tm.n_bits, r = t & rmask;
    long long so = inst * tm.bss;
    so += tm.tab[0][(int)((r >> 0) & 255)].src;
    so += tm.tab[1][(int)((r >> 8) & 255)].src;
    { const unsigned char* a_ = sthr + so + 0u; if ((((unsigned long long)a_) & 127ull) == 0) asm volatile("prefetch.global.L2 [%0];" :: "l"(a_)); }
    { const unsigned char* a_ = sthr + so + 131072u; if ((((unsigned long long)a_) & 127ull) == 0) asm volatile("prefetch.global.L2 [%0];" :: "l"(a_)); }
    { const unsigned char* a_ = sthr + so + 65536u; if ((((unsigned long long)a_) & 127ull) == 0) asm volatile("prefetch.global.L2 [%0];" :: "l"(a_)); }
    { const unsigned char* a_ = sthr + so + 196608u; if ((((unsigned long long)a_) & 127ull) == 0) asm volatile("prefetch.global.L2 [%0];" :: "l"(a_)); }
  } }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  for (long long t = t0 + gid; t < t1; t += n_groups) {
    const long long inst = t >> tm.n_bits, r = t & rmask;
    long long so = inst * tm.bss, dof = inst * tm.bsd;
    { const TileTab& e = tm.tab[0][(int)((r >> 0) & 255)]; so += e.src; dof += e.dst; }
    { const TileTab& e = tm.tab[1][(int)((r >> 8) & 255)]; so += e.src; dof += e.dst; }
    unsigned R[16], Q[16];
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(R[0]), "=r"(R[1]), "=r"(R[2]), "=r"(R[3]) : "l"(sthr + so + 0));
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(R[4]), "=r"(R[5]), "=r"(R[6]), "=r"(R[7]) : "l"(sthr + so + 131072));
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(R[8]), "=r"(R[9]), "=r"(R[10]), "=r"(R[11]) : "l"(sthr + so + 65536));
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(R[12]), "=r"(R[13]), "=r"(R[14]), "=r"(R[15]) : "l"(sthr + so + 196608));
  {
    unsigned T_[16];
    T_[0] = R[0];
    T_[1] = R[1];
    T_[2] = R[2];
    T_[3] = R[3];
    T_[4] = R[4];
    T_[5] = R[5];
    T_[6] = R[6];
    T_[7] = R[7];
    T_[8] = R[8];
    T_[9] = R[9];
    T_[10] = R[10];
    T_[11] = R[11];
    T_[12] = R[12];
    T_[13] = R[13];
    T_[14] = R[14];
    T_[15] = R[15];
    { const bool q_ = (fb >> 0) & 1;
      { unsigned x_ = T_[0], y_ = T_[1]; T_[0] = q_ ? y_ : x_; T_[1] = q_ ? x_ : y_; }
      { unsigned x_ = T_[2], y_ = T_[3]; T_[2] = q_ ? y_ : x_; T_[3] = q_ ? x_ : y_; }
      { unsigned x_ = T_[4], y_ = T_[5]; T_[4] = q_ ? y_ : x_; T_[5] = q_ ? x_ : y_; }
      { unsigned x_ = T_[6], y_ = T_[7]; T_[6] = q_ ? y_ : x_; T_[7] = q_ ? x_ : y_; }
      { unsigned x_ = T_[8], y_ = T_[9]; T_[8] = q_ ? y_ : x_; T_[9] = q_ ? x_ : y_; }
      { unsigned x_ = T_[10], y_ = T_[11]; T_[10] = q_ ? y_ : x_; T_[11] = q_ ? x_ : y_; }
      { unsigned x_ = T_[12], y_ = T_[13]; T_[12] = q_ ? y_ : x_; T_[13] = q_ ? x_ : y_; }
      { unsigned x_ = T_[14], y_ = T_[15]; T_[14] = q_ ? y_ : x_; T_[15] = q_ ? x_ : y_; }
    }
    { const bool q_ = (fb >> 1) & 1;
      { unsigned x_ = T_[0], y_ = T_[2]; T_[0] = q_ ? y_ : x_; T_[2] = q_ ? x_ : y_; }
      { unsigned x_ = T_[1], y_ = T_[3]; T_[1] = q_ ? y_ : x_; T_[3] = q_ ? x_ : y_; }
      { unsigned x_ = T_[4], y_ = T_[6]; T_[4] = q_ ? y_ : x_; T_[6] = q_ ? x_ : y_; }
      { unsigned x_ = T_[5], y_ = T_[7]; T_[5] = q_ ? y_ : x_; T_[7] = q_ ? x_ : y_; }
      { unsigned x_ = T_[8], y_ = T_[10]; T_[8] = q_ ? y_ : x_; T_[10] = q_ ? x_ : y_; }
      { unsigned x_ = T_[9], y_ = T_[11]; T_[9] = q_ ? y_ : x_; T_[11] = q_ ? x_ : y_; }
      { unsigned x_ = T_[12], y_ = T_[14]; T_[12] = q_ ? y_ : x_; T_[14] = q_ ? x_ : y_; }
      { unsigned x_ = T_[13], y_ = T_[15]; T_[13] = q_ ? y_ : x_; T_[15] = q_ ? x_ : y_; }
    }
    Q[0] = __shfl_sync(0xffffffffu, T_[0], 0 ^ fd);
    Q[1] = __shfl_sync(0xffffffffu, T_[1], 1 ^ fd);
    Q[2] = __shfl_sync(0xffffffffu, T_[2], 2 ^ fd);
    Q[3] = __shfl_sync(0xffffffffu, T_[3], 3 ^ fd);
    Q[8] = __shfl_sync(0xffffffffu, T_[8], 0 ^ fd);
    Q[9] = __shfl_sync(0xffffffffu, T_[9], 1 ^ fd);
    Q[10] = __shfl_sync(0xffffffffu, T_[10], 2 ^ fd);
    Q[11] = __shfl_sync(0xffffffffu, T_[11], 3 ^ fd);
    Q[4] = __shfl_sync(0xffffffffu, T_[4], 0 ^ fd);
    Q[5] = __shfl_sync(0xffffffffu, T_[5], 1 ^ fd);
    Q[6] = __shfl_sync(0xffffffffu, T_[6], 2 ^ fd);
    Q[7] = __shfl_sync(0xffffffffu, T_[7], 3 ^ fd);
    Q[12] = __shfl_sync(0xffffffffu, T_[12], 0 ^ fd);
    Q[13] = __shfl_sync(0xffffffffu, T_[13], 1 ^ fd);
    Q[14] = __shfl_sync(0xffffffffu, T_[14], 2 ^ fd);
    Q[15] = __shfl_sync(0xffffffffu, T_[15], 3 ^ fd);
    { const bool q_ = (fz >> 0) & 1;
      { unsigned x_ = Q[0], y_ = Q[1]; Q[0] = q_ ? y_ : x_; Q[1] = q_ ? x_ : y_; }
      { unsigned x_ = Q[2], y_ = Q[3]; Q[2] = q_ ? y_ : x_; Q[3] = q_ ? x_ : y_; }
      { unsigned x_ = Q[4], y_ = Q[5]; Q[4] = q_ ? y_ : x_; Q[5] = q_ ? x_ : y_; }
      { unsigned x_ = Q[6], y_ = Q[7]; Q[6] = q_ ? y_ : x_; Q[7] = q_ ? x_ : y_; }
      { unsigned x_ = Q[8], y_ = Q[9]; Q[8] = q_ ? y_ : x_; Q[9] = q_ ? x_ : y_; }
      { unsigned x_ = Q[10], y_ = Q[11]; Q[10] = q_ ? y_ : x_; Q[11] = q_ ? x_ : y_; }
      { unsigned x_ = Q[12], y_ = Q[13]; Q[12] = q_ ? y_ : x_; Q[13] = q_ ? x_ : y_; }
      { unsigned x_ = Q[14], y_ = Q[15]; Q[14] = q_ ? y_ : x_; Q[15] = q_ ? x_ : y_; }
    }
    { const bool q_ = (fz >> 1) & 1;
      { unsigned x_ = Q[0], y_ = Q[2]; Q[0] = q_ ? y_ : x_; Q[2] = q_ ? x_ : y_; }
      { unsigned x_ = Q[1], y_ = Q[3]; Q[1] = q_ ? y_ : x_; Q[3] = q_ ? x_ : y_; }
      { unsigned x_ = Q[4], y_ = Q[6]; Q[4] = q_ ? y_ : x_; Q[6] = q_ ? x_ : y_; }
      { unsigned x_ = Q[5], y_ = Q[7]; Q[5] = q_ ? y_ : x_; Q[7] = q_ ? x_ : y_; }
      { unsigned x_ = Q[8], y_ = Q[10]; Q[8] = q_ ? y_ : x_; Q[10] = q_ ? x_ : y_; }
      { unsigned x_ = Q[9], y_ = Q[11]; Q[9] = q_ ? y_ : x_; Q[11] = q_ ? x_ : y_; }
      { unsigned x_ = Q[12], y_ = Q[14]; Q[12] = q_ ? y_ : x_; Q[14] = q_ ? x_ : y_; }
      { unsigned x_ = Q[13], y_ = Q[15]; Q[13] = q_ ? y_ : x_; Q[15] = q_ ? x_ : y_; }
    }
  }
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(dthr + dof + 0), "r"(Q[0]), "r"(Q[1]), "r"(Q[2]), "r"(Q[3]) : "memory");
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(dthr + dof + 1024), "r"(Q[4]), "r"(Q[5]), "r"(Q[6]), "r"(Q[7]) : "memory");
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(dthr + dof + 512), "r"(Q[8]), "r"(Q[9]), "r"(Q[10]), "r"(Q[11]) : "memory");
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(dthr + dof + 1536), "r"(Q[12]), "r"(Q[13]), "r"(Q[14]), "r"(Q[15]) : "memory");
  }
}
