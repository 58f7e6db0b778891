struct TileTab { long long src, dst, sc; };
struct TileMap { long long n_tiles; int n_bits; int n_tab; long long bss, bsd; TileTab tab[3][256]; };
struct __align__(64) TMap { unsigned long long v[16]; };
__device__ __forceinline__ void mwait(unsigned b, unsigned ph) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" :: "r"(b), "r"(ph) : "memory");
}
extern "C" __global__ void __launch_bounds__(288, 1) ll_tma_hbm(
    const __grid_constant__ TileMap tm, const __grid_constant__ TMap tsrc,
    const __grid_constant__ TMap tdst, unsigned char* __restrict__ dst,
    long long t0, long long t1, long long src_shift, long long dst_shift) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ __align__(8) unsigned long long bars[6];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned sb = (((unsigned)__cvta_generic_to_shared(smem)) + 1023u) & ~1023u;
  const unsigned full0 = (unsigned)__cvta_generic_to_shared(bars), empty0 = full0 + 24u;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 3; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(full0 + 8 * i) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" :: "r"(empty0 + 8 * i) : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const long long rmask = (1LL << tm.n_bits) - 1;
  auto tile_off = [&](long long t, long long& so, long long& dof) {
    const long long inst = t >> tm.n_bits, r = t & rmask;
    so = inst * tm.bss; dof = inst * tm.bsd;
    { const TileTab& e = tm.tab[0][(int)((r >> 0) & 255)]; so += e.src; dof += e.dst; }
    { const TileTab& e = tm.tab[1][(int)((r >> 8) & 255)]; so += e.src; dof += e.dst; }
  };
  if (warp == 8) {
    if (lane == 0) {
      int s = 0; unsigned ph = 0;
      for (long long base = t0 + (long long)blockIdx.x * 1; base < t1; base += (long long)gridDim.x * 1) {
        { const long long t = base + 0; if (t < t1) {
          const unsigned fb = full0 + 8u * (s * 1 + 0), eb = empty0 + 8u * (s * 1 + 0);
          mwait(eb, ph ^ 1u);
          long long so, dof; tile_off(t, so, dof);
          const long long e = (so - src_shift) >> 1;
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(fb), "r"(32768u) : "memory");
          asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" :: "r"(sb + (unsigned)(s * 1 + 0) * 32768u), "l"(&tsrc), "r"((int)((e >> 0) & 8191LL)), "r"((int)((e >> 13))), "r"(fb) : "memory");
        } }
        if (++s == 3) { s = 0; ph ^= 1u; }
        if (base == t0 + (long long)blockIdx.x * 1) asm volatile("griddepcontrol.launch_dependents;");
      }
    }
    return;
  }
  const int g = warp >> 3;
  const int tb = lane | ((warp & 7) << 5);
  unsigned st_off = 0, srx = 0, swx = 0;
  if (tb & 1) { st_off += 0u; srx ^= 2064u; swx ^= 2064u; }
  if (tb & 2) { st_off += 0u; srx ^= 4128u; swx ^= 4128u; }
  if (tb & 4) { st_off += 0u; srx ^= 8256u; swx ^= 8256u; }
  if (tb & 8) { st_off += 0u; srx ^= 2048u; swx ^= 16u; }
  if (tb & 16) { st_off += 0u; srx ^= 4096u; swx ^= 32u; }
  if (tb & 32) { st_off += 0u; srx ^= 8192u; swx ^= 64u; }
  if (tb & 64) { st_off += 0u; srx ^= 16384u; swx ^= 128u; }
  if (tb & 128) { st_off += 0u; srx ^= 128u; swx ^= 16384u; }
  unsigned char* dthr = dst + st_off - dst_shift;
  (void)dthr; (void)swx;
  const unsigned db0 = sb + 3u * 32768u + (unsigned)g * 65536u;
  unsigned it = 0;
  int s = 0; unsigned ph = 0;
  for (long long t = t0 + (long long)blockIdx.x * 1 + g; t < t1; t += (long long)gridDim.x * 1) {
    const unsigned slot = (unsigned)(s * 1) + (unsigned)g;
    mwait(full0 + 8u * slot, ph);
    unsigned Q[32];
    const unsigned rb = sb + slot * 32768u;
    asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(Q[0]), "=r"(Q[1]), "=r"(Q[2]), "=r"(Q[3]) : "r"(rb + (srx ^ 0u)) : "memory");
    asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(Q[4]), "=r"(Q[5]), "=r"(Q[6]), "=r"(Q[7]) : "r"(rb + (srx ^ 256u)) : "memory");
    asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(Q[8]), "=r"(Q[9]), "=r"(Q[10]), "=r"(Q[11]) : "r"(rb + (srx ^ 512u)) : "memory");
    asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(Q[12]), "=r"(Q[13]), "=r"(Q[14]), "=r"(Q[15]) : "r"(rb + (srx ^ 768u)) : "memory");
    asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(Q[16]), "=r"(Q[17]), "=r"(Q[18]), "=r"(Q[19]) : "r"(rb + (srx ^ 1024u)) : "memory");
    asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(Q[20]), "=r"(Q[21]), "=r"(Q[22]), "=r"(Q[23]) : "r"(rb + (srx ^ 1280u)) : "memory");
    asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(Q[24]), "=r"(Q[25]), "=r"(Q[26]), "=r"(Q[27]) : "r"(rb + (srx ^ 1536u)) : "memory");
    asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(Q[28]), "=r"(Q[29]), "=r"(Q[30]), "=r"(Q[31]) : "r"(rb + (srx ^ 1792u)) : "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(empty0 + 8u * slot) : "memory");
  { unsigned x_ = Q[0], y_ = Q[4]; Q[0] = __byte_perm(x_, y_, 21520u); Q[4] = __byte_perm(x_, y_, 30258u); }
  { unsigned x_ = Q[1], y_ = Q[5]; Q[1] = __byte_perm(x_, y_, 21520u); Q[5] = __byte_perm(x_, y_, 30258u); }
  { unsigned x_ = Q[2], y_ = Q[6]; Q[2] = __byte_perm(x_, y_, 21520u); Q[6] = __byte_perm(x_, y_, 30258u); }
  { unsigned x_ = Q[3], y_ = Q[7]; Q[3] = __byte_perm(x_, y_, 21520u); Q[7] = __byte_perm(x_, y_, 30258u); }
  { unsigned x_ = Q[8], y_ = Q[12]; Q[8] = __byte_perm(x_, y_, 21520u); Q[12] = __byte_perm(x_, y_, 30258u); }
  { unsigned x_ = Q[9], y_ = Q[13]; Q[9] = __byte_perm(x_, y_, 21520u); Q[13] = __byte_perm(x_, y_, 30258u); }
  { unsigned x_ = Q[10], y_ = Q[14]; Q[10] = __byte_perm(x_, y_, 21520u); Q[14] = __byte_perm(x_, y_, 30258u); }
  { unsigned x_ = Q[11], y_ = Q[15]; Q[11] = __byte_perm(x_, y_, 21520u); Q[15] = __byte_perm(x_, y_, 30258u); }
  { unsigned x_ = Q[16], y_ = Q[20]; Q[16] = __byte_perm(x_, y_, 21520u); Q[20] = __byte_perm(x_, y_, 30258u); }
  { unsigned x_ = Q[17], y_ = Q[21]; Q[17] = __byte_perm(x_, y_, 21520u); Q[21] = __byte_perm(x_, y_, 30258u); }
  { unsigned x_ = Q[18], y_ = Q[22]; Q[18] = __byte_perm(x_, y_, 21520u); Q[22] = __byte_perm(x_, y_, 30258u); }
  { unsigned x_ = Q[19], y_ = Q[23]; Q[19] = __byte_perm(x_, y_, 21520u); Q[23] = __byte_perm(x_, y_, 30258u); }
  { unsigned x_ = Q[24], y_ = Q[28]; Q[24] = __byte_perm(x_, y_, 21520u); Q[28] = __byte_perm(x_, y_, 30258u); }
  { unsigned x_ = Q[25], y_ = Q[29]; Q[25] = __byte_perm(x_, y_, 21520u); Q[29] = __byte_perm(x_, y_, 30258u); }
  { unsigned x_ = Q[26], y_ = Q[30]; Q[26] = __byte_perm(x_, y_, 21520u); Q[30] = __byte_perm(x_, y_, 30258u); }
  { unsigned x_ = Q[27], y_ = Q[31]; Q[27] = __byte_perm(x_, y_, 21520u); Q[31] = __byte_perm(x_, y_, 30258u); }
    long long so, dof; tile_off(t, so, dof);
    const unsigned db = db0 + (it & 1u) * 32768u;
    if (tb == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    asm volatile("bar.sync %0, %1;" :: "r"(g + 1), "r"(256) : "memory");
    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" :: "r"(db + (swx ^ 0u)), "r"(Q[0]), "r"(Q[8]), "r"(Q[16]), "r"(Q[24]) : "memory");
    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" :: "r"(db + (swx ^ 512u)), "r"(Q[1]), "r"(Q[9]), "r"(Q[17]), "r"(Q[25]) : "memory");
    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" :: "r"(db + (swx ^ 1024u)), "r"(Q[2]), "r"(Q[10]), "r"(Q[18]), "r"(Q[26]) : "memory");
    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" :: "r"(db + (swx ^ 1536u)), "r"(Q[3]), "r"(Q[11]), "r"(Q[19]), "r"(Q[27]) : "memory");
    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" :: "r"(db + (swx ^ 256u)), "r"(Q[4]), "r"(Q[12]), "r"(Q[20]), "r"(Q[28]) : "memory");
    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" :: "r"(db + (swx ^ 768u)), "r"(Q[5]), "r"(Q[13]), "r"(Q[21]), "r"(Q[29]) : "memory");
    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" :: "r"(db + (swx ^ 1280u)), "r"(Q[6]), "r"(Q[14]), "r"(Q[22]), "r"(Q[30]) : "memory");
    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" :: "r"(db + (swx ^ 1792u)), "r"(Q[7]), "r"(Q[15]), "r"(Q[23]), "r"(Q[31]) : "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("bar.sync %0, %1;" :: "r"(g + 1), "r"(256) : "memory");
    if (tb == 0) {
      const long long e = (dof - dst_shift) >> 1;
      asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" :: "l"(&tdst), "r"((int)((e >> 0) & 8191LL)), "r"((int)((e >> 13))), "r"(db) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    ++it;
    if (++s == 3) { s = 0; ph ^= 1u; }
  }
  if (tb == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
