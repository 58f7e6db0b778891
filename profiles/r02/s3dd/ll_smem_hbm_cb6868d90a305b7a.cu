struct TileTab { long long src, dst, sc; };
struct TileMap { long long n_tiles; int n_bits; int n_tab; long long bss, bsd; TileTab tab[3][256]; };
extern "C" __global__ void __launch_bounds__(256, 4) ll_smem_hbm(
    const __grid_constant__ TileMap tm, const unsigned char* __restrict__ src,
    unsigned char* __restrict__ dst, long long n_groups, long long t0, long long t1,
    long long src_shift, long long dst_shift, long long pf_ctas) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int group = warp >> 0;
  const int tb = lane | ((warp & 0) << 5);
  const long long gid = (long long)blockIdx.x * 8 + group;
  if (gid >= n_groups) return;
  unsigned ld_off = 0, st_off = 0, swx = 0, srx = 0;
  if (tb & 1) { ld_off += 16u; st_off += 16u; swx ^= 320u; srx ^= 16u; }
  if (tb & 2) { ld_off += 32u; st_off += 32u; swx ^= 32u; srx ^= 32u; }
  if (tb & 4) { ld_off += 64u; st_off += 64u; swx ^= 8u; srx ^= 136u; }
  if (tb & 8) { ld_off += 128u; st_off += 128u; swx ^= 16u; srx ^= 64u; }
  if (tb & 16) { ld_off += 256u; st_off += 256u; swx ^= 512u; srx ^= 512u; }
  const unsigned char* sthr = src + ld_off - src_shift;
  unsigned char* dthr = dst + st_off - dst_shift;
  const long long rmask = (1LL << tm.n_bits) - 1;
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(smem) + group * 4096u;
  unsigned buf = 0;
  unsigned R[16], Q[16];
  long long so = 0, dof = 0;
  auto tile_off = [&](long long t) {
    const long long inst = t >> tm.n_bits;
    long long r = t & rmask;
    so = inst * tm.bss; dof = inst * tm.bsd;
    { const TileTab& e = tm.tab[0][(int)((r >> 0) & 255)]; so += e.src; dof += e.dst; }
    { const TileTab& e = tm.tab[1][(int)((r >> 8) & 255)]; so += e.src; dof += e.dst; }
    { const TileTab& e = tm.tab[2][(int)((r >> 16) & 255)]; so += e.src; dof += e.dst; }
  };
  { const long long tp = t0 + gid + 0LL * pf_ctas * 8; if (tp < t1 && blockIdx.x < pf_ctas) { tile_off(tp);
    { const unsigned char* a_ = sthr + so + 0u; if ((((unsigned long long)a_) & 127ull) == 0) asm volatile("cp.async.bulk.prefetch.L2.global [%0], 128;" :: "l"(a_)); }
    { const unsigned char* a_ = sthr + so + 2048u; if ((((unsigned long long)a_) & 127ull) == 0) asm volatile("cp.async.bulk.prefetch.L2.global [%0], 128;" :: "l"(a_)); }
    { const unsigned char* a_ = sthr + so + 512u; if ((((unsigned long long)a_) & 127ull) == 0) asm volatile("cp.async.bulk.prefetch.L2.global [%0], 128;" :: "l"(a_)); }
    { const unsigned char* a_ = sthr + so + 2560u; if ((((unsigned long long)a_) & 127ull) == 0) asm volatile("cp.async.bulk.prefetch.L2.global [%0], 128;" :: "l"(a_)); }
  } }
  { const long long tp = t0 + gid + 1LL * pf_ctas * 8; if (tp < t1 && blockIdx.x < pf_ctas) { tile_off(tp);
    { const unsigned char* a_ = sthr + so + 0u; if ((((unsigned long long)a_) & 127ull) == 0) asm volatile("cp.async.bulk.prefetch.L2.global [%0], 128;" :: "l"(a_)); }
    { const unsigned char* a_ = sthr + so + 2048u; if ((((unsigned long long)a_) & 127ull) == 0) asm volatile("cp.async.bulk.prefetch.L2.global [%0], 128;" :: "l"(a_)); }
    { const unsigned char* a_ = sthr + so + 512u; if ((((unsigned long long)a_) & 127ull) == 0) asm volatile("cp.async.bulk.prefetch.L2.global [%0], 128;" :: "l"(a_)); }
    { const unsigned char* a_ = sthr + so + 2560u; if ((((unsigned long long)a_) & 127ull) == 0) asm volatile("cp.async.bulk.prefetch.L2.global [%0], 128;" :: "l"(a_)); }
  } }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  long long t = t0 + gid;
  long long da = 0;
  if (t < t1) { tile_off(t); da = dof;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(R[0]), "=r"(R[1]), "=r"(R[2]), "=r"(R[3]) : "l"(sthr + so + 0));
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(R[4]), "=r"(R[5]), "=r"(R[6]), "=r"(R[7]) : "l"(sthr + so + 2048));
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(R[8]), "=r"(R[9]), "=r"(R[10]), "=r"(R[11]) : "l"(sthr + so + 512));
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(R[12]), "=r"(R[13]), "=r"(R[14]), "=r"(R[15]) : "l"(sthr + so + 2560));
  }
  asm volatile("griddepcontrol.launch_dependents;");
  for (; t < t1; t += n_groups) {
    { const long long dcur = da;
  { unsigned x_ = R[0], y_ = R[4]; R[0] = __byte_perm(x_, y_, 25152u); R[4] = __byte_perm(x_, y_, 29521u); }
  { unsigned x_ = R[1], y_ = R[5]; R[1] = __byte_perm(x_, y_, 25152u); R[5] = __byte_perm(x_, y_, 29521u); }
  { unsigned x_ = R[2], y_ = R[6]; R[2] = __byte_perm(x_, y_, 25152u); R[6] = __byte_perm(x_, y_, 29521u); }
  { unsigned x_ = R[3], y_ = R[7]; R[3] = __byte_perm(x_, y_, 25152u); R[7] = __byte_perm(x_, y_, 29521u); }
  { unsigned x_ = R[8], y_ = R[12]; R[8] = __byte_perm(x_, y_, 25152u); R[12] = __byte_perm(x_, y_, 29521u); }
  { unsigned x_ = R[9], y_ = R[13]; R[9] = __byte_perm(x_, y_, 25152u); R[13] = __byte_perm(x_, y_, 29521u); }
  { unsigned x_ = R[10], y_ = R[14]; R[10] = __byte_perm(x_, y_, 25152u); R[14] = __byte_perm(x_, y_, 29521u); }
  { unsigned x_ = R[11], y_ = R[15]; R[11] = __byte_perm(x_, y_, 25152u); R[15] = __byte_perm(x_, y_, 29521u); }
  { unsigned x_ = R[0], y_ = R[1]; R[0] = __byte_perm(x_, y_, 21520u); R[1] = __byte_perm(x_, y_, 30258u); }
  { unsigned x_ = R[2], y_ = R[3]; R[2] = __byte_perm(x_, y_, 21520u); R[3] = __byte_perm(x_, y_, 30258u); }
  { unsigned x_ = R[4], y_ = R[5]; R[4] = __byte_perm(x_, y_, 21520u); R[5] = __byte_perm(x_, y_, 30258u); }
  { unsigned x_ = R[6], y_ = R[7]; R[6] = __byte_perm(x_, y_, 21520u); R[7] = __byte_perm(x_, y_, 30258u); }
  { unsigned x_ = R[8], y_ = R[9]; R[8] = __byte_perm(x_, y_, 21520u); R[9] = __byte_perm(x_, y_, 30258u); }
  { unsigned x_ = R[10], y_ = R[11]; R[10] = __byte_perm(x_, y_, 21520u); R[11] = __byte_perm(x_, y_, 30258u); }
  { unsigned x_ = R[12], y_ = R[13]; R[12] = __byte_perm(x_, y_, 21520u); R[13] = __byte_perm(x_, y_, 30258u); }
  { unsigned x_ = R[14], y_ = R[15]; R[14] = __byte_perm(x_, y_, 21520u); R[15] = __byte_perm(x_, y_, 30258u); }
    asm volatile("st.shared.v2.b32 [%0], {%1,%2};" :: "r"(sbase + buf + (swx ^ 0u)), "r"(R[0]), "r"(R[2]) : "memory");
    asm volatile("st.shared.v2.b32 [%0], {%1,%2};" :: "r"(sbase + buf + (swx ^ 64u)), "r"(R[1]), "r"(R[3]) : "memory");
    asm volatile("st.shared.v2.b32 [%0], {%1,%2};" :: "r"(sbase + buf + (swx ^ 136u)), "r"(R[4]), "r"(R[6]) : "memory");
    asm volatile("st.shared.v2.b32 [%0], {%1,%2};" :: "r"(sbase + buf + (swx ^ 200u)), "r"(R[5]), "r"(R[7]) : "memory");
    asm volatile("st.shared.v2.b32 [%0], {%1,%2};" :: "r"(sbase + buf + (swx ^ 1024u)), "r"(R[8]), "r"(R[10]) : "memory");
    asm volatile("st.shared.v2.b32 [%0], {%1,%2};" :: "r"(sbase + buf + (swx ^ 1088u)), "r"(R[9]), "r"(R[11]) : "memory");
    asm volatile("st.shared.v2.b32 [%0], {%1,%2};" :: "r"(sbase + buf + (swx ^ 1160u)), "r"(R[12]), "r"(R[14]) : "memory");
    asm volatile("st.shared.v2.b32 [%0], {%1,%2};" :: "r"(sbase + buf + (swx ^ 1224u)), "r"(R[13]), "r"(R[15]) : "memory");
    { const long long tn = t + 1 * n_groups; if (tn < t1) { tile_off(tn); da = dof;
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(R[0]), "=r"(R[1]), "=r"(R[2]), "=r"(R[3]) : "l"(sthr + so + 0));
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(R[4]), "=r"(R[5]), "=r"(R[6]), "=r"(R[7]) : "l"(sthr + so + 2048));
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(R[8]), "=r"(R[9]), "=r"(R[10]), "=r"(R[11]) : "l"(sthr + so + 512));
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(R[12]), "=r"(R[13]), "=r"(R[14]), "=r"(R[15]) : "l"(sthr + so + 2560));
    } }
    __syncwarp();
    asm volatile("ld.shared.v2.b32 {%0,%1}, [%2];" : "=r"(Q[0]), "=r"(Q[1]) : "r"(sbase + buf + (srx ^ 0u)) : "memory");
    asm volatile("ld.shared.v2.b32 {%0,%1}, [%2];" : "=r"(Q[2]), "=r"(Q[3]) : "r"(sbase + buf + (srx ^ 8u)) : "memory");
    asm volatile("ld.shared.v2.b32 {%0,%1}, [%2];" : "=r"(Q[4]), "=r"(Q[5]) : "r"(sbase + buf + (srx ^ 320u)) : "memory");
    asm volatile("ld.shared.v2.b32 {%0,%1}, [%2];" : "=r"(Q[6]), "=r"(Q[7]) : "r"(sbase + buf + (srx ^ 328u)) : "memory");
    asm volatile("ld.shared.v2.b32 {%0,%1}, [%2];" : "=r"(Q[8]), "=r"(Q[9]) : "r"(sbase + buf + (srx ^ 1024u)) : "memory");
    asm volatile("ld.shared.v2.b32 {%0,%1}, [%2];" : "=r"(Q[10]), "=r"(Q[11]) : "r"(sbase + buf + (srx ^ 1032u)) : "memory");
    asm volatile("ld.shared.v2.b32 {%0,%1}, [%2];" : "=r"(Q[12]), "=r"(Q[13]) : "r"(sbase + buf + (srx ^ 1344u)) : "memory");
    asm volatile("ld.shared.v2.b32 {%0,%1}, [%2];" : "=r"(Q[14]), "=r"(Q[15]) : "r"(sbase + buf + (srx ^ 1352u)) : "memory");
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(dthr + dcur + 0), "r"(Q[0]), "r"(Q[1]), "r"(Q[2]), "r"(Q[3]) : "memory");
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(dthr + dcur + 4096), "r"(Q[4]), "r"(Q[5]), "r"(Q[6]), "r"(Q[7]) : "memory");
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(dthr + dcur + 512), "r"(Q[8]), "r"(Q[9]), "r"(Q[10]), "r"(Q[11]) : "memory");
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(dthr + dcur + 4608), "r"(Q[12]), "r"(Q[13]), "r"(Q[14]), "r"(Q[15]) : "memory");
    buf ^= 2048u; }
  }
}
