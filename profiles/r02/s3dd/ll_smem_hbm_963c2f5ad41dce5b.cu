struct TileTab { long long src, dst, sc; };
struct TileMap { long long n_tiles; int n_bits; int n_tab; long long bss, bsd; TileTab tab[3][256]; };
extern "C" __global__ void __launch_bounds__(256, 3) ll_smem_hbm(
    const __grid_constant__ TileMap tm, const unsigned char* __restrict__ src,
    unsigned char* __restrict__ dst, long long n_groups, long long t0, long long t1,
    long long src_shift, long long dst_shift, long long pf_ctas) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int group = warp >> 1;
  const int tb = lane | ((warp & 1) << 5);
  const long long gid = (long long)blockIdx.x * 4 + group;
  if (gid >= n_groups) return;
  unsigned ld_off = 0, st_off = 0, swx = 0, srx = 0;
  if (tb & 1) { ld_off += 16u; st_off += 16u; swx ^= 144u; srx ^= 16u; }
  if (tb & 2) { ld_off += 32u; st_off += 32u; swx ^= 288u; srx ^= 32u; }
  if (tb & 4) { ld_off += 64u; st_off += 16384u; swx ^= 576u; srx ^= 64u; }
  if (tb & 8) { ld_off += 128u; st_off += 32768u; swx ^= 4096u; srx ^= 1024u; }
  if (tb & 16) { ld_off += 131072u; st_off += 65536u; swx ^= 16u; srx ^= 2048u; }
  if (tb & 32) { ld_off += 262144u; st_off += 131072u; swx ^= 32u; srx ^= 144u; }
  const unsigned char* sthr = src + ld_off - src_shift;
  unsigned char* dthr = dst + st_off - dst_shift;
  const long long rmask = (1LL << tm.n_bits) - 1;
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(smem) + group * 16384u;
  unsigned buf = 0;
  unsigned R[32], Q[32];
  long long so = 0, dof = 0;
  auto tile_off = [&](long long t) {
    const long long inst = t >> tm.n_bits;
    long long r = t & rmask;
    so = inst * tm.bss; dof = inst * tm.bsd;
    { const TileTab& e = tm.tab[0][(int)((r >> 0) & 255)]; so += e.src; dof += e.dst; }
    { const TileTab& e = tm.tab[1][(int)((r >> 8) & 255)]; so += e.src; dof += e.dst; }
  };
  { const long long tp = t0 + gid + 0LL * pf_ctas * 4; if (tp < t1 && blockIdx.x < pf_ctas) { tile_off(tp);
    { const unsigned char* a_ = sthr + so + 0u; if ((((unsigned long long)a_) & 127ull) == 0) asm volatile("cp.async.bulk.prefetch.L2.global [%0], 128;" :: "l"(a_)); }
    { const unsigned char* a_ = sthr + so + 16384u; if ((((unsigned long long)a_) & 127ull) == 0) asm volatile("cp.async.bulk.prefetch.L2.global [%0], 128;" :: "l"(a_)); }
    { const unsigned char* a_ = sthr + so + 32768u; if ((((unsigned long long)a_) & 127ull) == 0) asm volatile("cp.async.bulk.prefetch.L2.global [%0], 128;" :: "l"(a_)); }
    { const unsigned char* a_ = sthr + so + 49152u; if ((((unsigned long long)a_) & 127ull) == 0) asm volatile("cp.async.bulk.prefetch.L2.global [%0], 128;" :: "l"(a_)); }
    { const unsigned char* a_ = sthr + so + 65536u; if ((((unsigned long long)a_) & 127ull) == 0) asm volatile("cp.async.bulk.prefetch.L2.global [%0], 128;" :: "l"(a_)); }
    { const unsigned char* a_ = sthr + so + 81920u; if ((((unsigned long long)a_) & 127ull) == 0) asm volatile("cp.async.bulk.prefetch.L2.global [%0], 128;" :: "l"(a_)); }
    { const unsigned char* a_ = sthr + so + 98304u; if ((((unsigned long long)a_) & 127ull) == 0) asm volatile("cp.async.bulk.prefetch.L2.global [%0], 128;" :: "l"(a_)); }
    { const unsigned char* a_ = sthr + so + 114688u; if ((((unsigned long long)a_) & 127ull) == 0) asm volatile("cp.async.bulk.prefetch.L2.global [%0], 128;" :: "l"(a_)); }
  } }
  { const long long tp = t0 + gid + 1LL * pf_ctas * 4; if (tp < t1 && blockIdx.x < pf_ctas) { tile_off(tp);
    { const unsigned char* a_ = sthr + so + 0u; if ((((unsigned long long)a_) & 127ull) == 0) asm volatile("cp.async.bulk.prefetch.L2.global [%0], 128;" :: "l"(a_)); }
    { const unsigned char* a_ = sthr + so + 16384u; if ((((unsigned long long)a_) & 127ull) == 0) asm volatile("cp.async.bulk.prefetch.L2.global [%0], 128;" :: "l"(a_)); }
    { const unsigned char* a_ = sthr + so + 32768u; if ((((unsigned long long)a_) & 127ull) == 0) asm volatile("cp.async.bulk.prefetch.L2.global [%0], 128;" :: "l"(a_)); }
    { const unsigned char* a_ = sthr + so + 49152u; if ((((unsigned long long)a_) & 127ull) == 0) asm volatile("cp.async.bulk.prefetch.L2.global [%0], 128;" :: "l"(a_)); }
    { const unsigned char* a_ = sthr + so + 65536u; if ((((unsigned long long)a_) & 127ull) == 0) asm volatile("cp.async.bulk.prefetch.L2.global [%0], 128;" :: "l"(a_)); }
    { const unsigned char* a_ = sthr + so + 81920u; if ((((unsigned long long)a_) & 127ull) == 0) asm volatile("cp.async.bulk.prefetch.L2.global [%0], 128;" :: "l"(a_)); }
    { const unsigned char* a_ = sthr + so + 98304u; if ((((unsigned long long)a_) & 127ull) == 0) asm volatile("cp.async.bulk.prefetch.L2.global [%0], 128;" :: "l"(a_)); }
    { const unsigned char* a_ = sthr + so + 114688u; if ((((unsigned long long)a_) & 127ull) == 0) asm volatile("cp.async.bulk.prefetch.L2.global [%0], 128;" :: "l"(a_)); }
  } }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  long long t = t0 + gid;
  long long da = 0;
  if (t < t1) { tile_off(t); da = dof;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(R[0]), "=r"(R[1]), "=r"(R[2]), "=r"(R[3]) : "l"(sthr + so + 0));
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(R[4]), "=r"(R[5]), "=r"(R[6]), "=r"(R[7]) : "l"(sthr + so + 16384));
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(R[8]), "=r"(R[9]), "=r"(R[10]), "=r"(R[11]) : "l"(sthr + so + 32768));
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(R[12]), "=r"(R[13]), "=r"(R[14]), "=r"(R[15]) : "l"(sthr + so + 49152));
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(R[16]), "=r"(R[17]), "=r"(R[18]), "=r"(R[19]) : "l"(sthr + so + 65536));
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(R[20]), "=r"(R[21]), "=r"(R[22]), "=r"(R[23]) : "l"(sthr + so + 81920));
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(R[24]), "=r"(R[25]), "=r"(R[26]), "=r"(R[27]) : "l"(sthr + so + 98304));
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(R[28]), "=r"(R[29]), "=r"(R[30]), "=r"(R[31]) : "l"(sthr + so + 114688));
  }
  asm volatile("griddepcontrol.launch_dependents;");
  for (; t < t1; t += n_groups) {
    { const long long dcur = da;
  { unsigned x_ = R[0], y_ = R[4]; R[0] = __byte_perm(x_, y_, 21520u); R[4] = __byte_perm(x_, y_, 30258u); }
  { unsigned x_ = R[1], y_ = R[5]; R[1] = __byte_perm(x_, y_, 21520u); R[5] = __byte_perm(x_, y_, 30258u); }
  { unsigned x_ = R[2], y_ = R[6]; R[2] = __byte_perm(x_, y_, 21520u); R[6] = __byte_perm(x_, y_, 30258u); }
  { unsigned x_ = R[3], y_ = R[7]; R[3] = __byte_perm(x_, y_, 21520u); R[7] = __byte_perm(x_, y_, 30258u); }
  { unsigned x_ = R[8], y_ = R[12]; R[8] = __byte_perm(x_, y_, 21520u); R[12] = __byte_perm(x_, y_, 30258u); }
  { unsigned x_ = R[9], y_ = R[13]; R[9] = __byte_perm(x_, y_, 21520u); R[13] = __byte_perm(x_, y_, 30258u); }
  { unsigned x_ = R[10], y_ = R[14]; R[10] = __byte_perm(x_, y_, 21520u); R[14] = __byte_perm(x_, y_, 30258u); }
  { unsigned x_ = R[11], y_ = R[15]; R[11] = __byte_perm(x_, y_, 21520u); R[15] = __byte_perm(x_, y_, 30258u); }
  { unsigned x_ = R[16], y_ = R[20]; R[16] = __byte_perm(x_, y_, 21520u); R[20] = __byte_perm(x_, y_, 30258u); }
  { unsigned x_ = R[17], y_ = R[21]; R[17] = __byte_perm(x_, y_, 21520u); R[21] = __byte_perm(x_, y_, 30258u); }
  { unsigned x_ = R[18], y_ = R[22]; R[18] = __byte_perm(x_, y_, 21520u); R[22] = __byte_perm(x_, y_, 30258u); }
  { unsigned x_ = R[19], y_ = R[23]; R[19] = __byte_perm(x_, y_, 21520u); R[23] = __byte_perm(x_, y_, 30258u); }
  { unsigned x_ = R[24], y_ = R[28]; R[24] = __byte_perm(x_, y_, 21520u); R[28] = __byte_perm(x_, y_, 30258u); }
  { unsigned x_ = R[25], y_ = R[29]; R[25] = __byte_perm(x_, y_, 21520u); R[29] = __byte_perm(x_, y_, 30258u); }
  { unsigned x_ = R[26], y_ = R[30]; R[26] = __byte_perm(x_, y_, 21520u); R[30] = __byte_perm(x_, y_, 30258u); }
  { unsigned x_ = R[27], y_ = R[31]; R[27] = __byte_perm(x_, y_, 21520u); R[31] = __byte_perm(x_, y_, 30258u); }
    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" :: "r"(sbase + buf + (swx ^ 0u)), "r"(R[0]), "r"(R[8]), "r"(R[16]), "r"(R[24]) : "memory");
    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" :: "r"(sbase + buf + (swx ^ 1024u)), "r"(R[1]), "r"(R[9]), "r"(R[17]), "r"(R[25]) : "memory");
    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" :: "r"(sbase + buf + (swx ^ 2048u)), "r"(R[2]), "r"(R[10]), "r"(R[18]), "r"(R[26]) : "memory");
    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" :: "r"(sbase + buf + (swx ^ 3072u)), "r"(R[3]), "r"(R[11]), "r"(R[19]), "r"(R[27]) : "memory");
    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" :: "r"(sbase + buf + (swx ^ 64u)), "r"(R[4]), "r"(R[12]), "r"(R[20]), "r"(R[28]) : "memory");
    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" :: "r"(sbase + buf + (swx ^ 1088u)), "r"(R[5]), "r"(R[13]), "r"(R[21]), "r"(R[29]) : "memory");
    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" :: "r"(sbase + buf + (swx ^ 2112u)), "r"(R[6]), "r"(R[14]), "r"(R[22]), "r"(R[30]) : "memory");
    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" :: "r"(sbase + buf + (swx ^ 3136u)), "r"(R[7]), "r"(R[15]), "r"(R[23]), "r"(R[31]) : "memory");
    { const long long tn = t + 1 * n_groups; if (tn < t1) { tile_off(tn); da = dof;
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(R[0]), "=r"(R[1]), "=r"(R[2]), "=r"(R[3]) : "l"(sthr + so + 0));
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(R[4]), "=r"(R[5]), "=r"(R[6]), "=r"(R[7]) : "l"(sthr + so + 16384));
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(R[8]), "=r"(R[9]), "=r"(R[10]), "=r"(R[11]) : "l"(sthr + so + 32768));
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(R[12]), "=r"(R[13]), "=r"(R[14]), "=r"(R[15]) : "l"(sthr + so + 49152));
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(R[16]), "=r"(R[17]), "=r"(R[18]), "=r"(R[19]) : "l"(sthr + so + 65536));
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(R[20]), "=r"(R[21]), "=r"(R[22]), "=r"(R[23]) : "l"(sthr + so + 81920));
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(R[24]), "=r"(R[25]), "=r"(R[26]), "=r"(R[27]) : "l"(sthr + so + 98304));
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(R[28]), "=r"(R[29]), "=r"(R[30]), "=r"(R[31]) : "l"(sthr + so + 114688));
    } }
    asm volatile("bar.sync %0, %1;" :: "r"(group + 1), "r"(64) : "memory");
    asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(Q[0]), "=r"(Q[1]), "=r"(Q[2]), "=r"(Q[3]) : "r"(sbase + buf + (srx ^ 0u)) : "memory");
    asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(Q[4]), "=r"(Q[5]), "=r"(Q[6]), "=r"(Q[7]) : "r"(sbase + buf + (srx ^ 4096u)) : "memory");
    asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(Q[8]), "=r"(Q[9]), "=r"(Q[10]), "=r"(Q[11]) : "r"(sbase + buf + (srx ^ 576u)) : "memory");
    asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(Q[12]), "=r"(Q[13]), "=r"(Q[14]), "=r"(Q[15]) : "r"(sbase + buf + (srx ^ 4672u)) : "memory");
    asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(Q[16]), "=r"(Q[17]), "=r"(Q[18]), "=r"(Q[19]) : "r"(sbase + buf + (srx ^ 288u)) : "memory");
    asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(Q[20]), "=r"(Q[21]), "=r"(Q[22]), "=r"(Q[23]) : "r"(sbase + buf + (srx ^ 4384u)) : "memory");
    asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(Q[24]), "=r"(Q[25]), "=r"(Q[26]), "=r"(Q[27]) : "r"(sbase + buf + (srx ^ 864u)) : "memory");
    asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(Q[28]), "=r"(Q[29]), "=r"(Q[30]), "=r"(Q[31]) : "r"(sbase + buf + (srx ^ 4960u)) : "memory");
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(dthr + dcur + 0), "r"(Q[0]), "r"(Q[1]), "r"(Q[2]), "r"(Q[3]) : "memory");
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(dthr + dcur + 1048576), "r"(Q[4]), "r"(Q[5]), "r"(Q[6]), "r"(Q[7]) : "memory");
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(dthr + dcur + 524288), "r"(Q[8]), "r"(Q[9]), "r"(Q[10]), "r"(Q[11]) : "memory");
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(dthr + dcur + 1572864), "r"(Q[12]), "r"(Q[13]), "r"(Q[14]), "r"(Q[15]) : "memory");
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(dthr + dcur + 262144), "r"(Q[16]), "r"(Q[17]), "r"(Q[18]), "r"(Q[19]) : "memory");
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(dthr + dcur + 1310720), "r"(Q[20]), "r"(Q[21]), "r"(Q[22]), "r"(Q[23]) : "memory");
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(dthr + dcur + 786432), "r"(Q[24]), "r"(Q[25]), "r"(Q[26]), "r"(Q[27]) : "memory");
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(dthr + dcur + 1835008), "r"(Q[28]), "r"(Q[29]), "r"(Q[30]), "r"(Q[31]) : "memory");
    buf ^= 8192u; }
  }
}
