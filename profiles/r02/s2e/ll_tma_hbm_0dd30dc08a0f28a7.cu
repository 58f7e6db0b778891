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
  __shared__ __align__(8) unsigned long long bars[12];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned sb = (((unsigned)__cvta_generic_to_shared(smem)) + 1023u) & ~1023u;
  const unsigned full0 = (unsigned)__cvta_generic_to_shared(bars), empty0 = full0 + 48u;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 6; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(full0 + 8 * i) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 4;" :: "r"(empty0 + 8 * i) : "memory");
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
      for (long long base = t0 + (long long)blockIdx.x * 2; base < t1; base += (long long)gridDim.x * 2) {
        { const long long t = base + 0; if (t < t1) {
          const unsigned fb = full0 + 8u * (s * 2 + 0), eb = empty0 + 8u * (s * 2 + 0);
          mwait(eb, ph ^ 1u);
          long long so, dof; tile_off(t, so, dof);
          const long long e = (so - src_shift) >> 1;
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(fb), "r"(8192u) : "memory");
          asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" :: "r"(sb + (unsigned)(s * 2 + 0) * 8192u), "l"(&tsrc), "r"((int)((e >> 0) & 255LL)), "r"((int)((e >> 8) & 15LL)), "r"((int)((e >> 12))), "r"(fb) : "memory");
        } }
        { const long long t = base + 1; if (t < t1) {
          const unsigned fb = full0 + 8u * (s * 2 + 1), eb = empty0 + 8u * (s * 2 + 1);
          mwait(eb, ph ^ 1u);
          long long so, dof; tile_off(t, so, dof);
          const long long e = (so - src_shift) >> 1;
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(fb), "r"(8192u) : "memory");
          asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" :: "r"(sb + (unsigned)(s * 2 + 1) * 8192u), "l"(&tsrc), "r"((int)((e >> 0) & 255LL)), "r"((int)((e >> 8) & 15LL)), "r"((int)((e >> 12))), "r"(fb) : "memory");
        } }
        if (++s == 3) { s = 0; ph ^= 1u; }
        if (base == t0 + (long long)blockIdx.x * 2) asm volatile("griddepcontrol.launch_dependents;");
      }
    }
    return;
  }
  const int g = warp >> 2;
  const int tb = lane | ((warp & 3) << 5);
  unsigned st_off = 0, srx = 0, swx = 0;
  if (tb & 1) { st_off += 0u; srx ^= 16u; swx ^= 576u; }
  if (tb & 2) { st_off += 0u; srx ^= 160u; swx ^= 1056u; }
  if (tb & 4) { st_off += 0u; srx ^= 4160u; swx ^= 2192u; }
  if (tb & 8) { st_off += 0u; srx ^= 128u; swx ^= 32u; }
  if (tb & 16) { st_off += 0u; srx ^= 2048u; swx ^= 64u; }
  if (tb & 32) { st_off += 0u; srx ^= 4096u; swx ^= 144u; }
  if (tb & 64) { st_off += 0u; srx ^= 1024u; swx ^= 4096u; }
  unsigned char* dthr = dst + st_off - dst_shift;
  (void)dthr; (void)swx;
  const unsigned db0 = sb + 6u * 8192u + (unsigned)g * 16384u;
  unsigned it = 0;
  int s = 0; unsigned ph = 0;
  for (long long t = t0 + (long long)blockIdx.x * 2 + g; t < t1; t += (long long)gridDim.x * 2) {
    const unsigned slot = (unsigned)(s * 2) + (unsigned)g;
    mwait(full0 + 8u * slot, ph);
    unsigned Q[16];
    const unsigned rb = sb + slot * 8192u;
    asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(Q[0]), "=r"(Q[1]), "=r"(Q[2]), "=r"(Q[3]) : "r"(rb + (srx ^ 0u)) : "memory");
    asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(Q[4]), "=r"(Q[5]), "=r"(Q[6]), "=r"(Q[7]) : "r"(rb + (srx ^ 256u)) : "memory");
    asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(Q[8]), "=r"(Q[9]), "=r"(Q[10]), "=r"(Q[11]) : "r"(rb + (srx ^ 512u)) : "memory");
    asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(Q[12]), "=r"(Q[13]), "=r"(Q[14]), "=r"(Q[15]) : "r"(rb + (srx ^ 768u)) : "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(empty0 + 8u * slot) : "memory");
    long long so, dof; tile_off(t, so, dof);
    const unsigned db = db0 + (it & 1u) * 8192u;
    if (tb == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    asm volatile("bar.sync %0, %1;" :: "r"(g + 1), "r"(128) : "memory");
    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" :: "r"(db + (swx ^ 0u)), "r"(Q[0]), "r"(Q[4]), "r"(Q[8]), "r"(Q[12]) : "memory");
    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" :: "r"(db + (swx ^ 16u)), "r"(Q[1]), "r"(Q[5]), "r"(Q[9]), "r"(Q[13]) : "memory");
    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" :: "r"(db + (swx ^ 288u)), "r"(Q[2]), "r"(Q[6]), "r"(Q[10]), "r"(Q[14]) : "memory");
    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" :: "r"(db + (swx ^ 304u)), "r"(Q[3]), "r"(Q[7]), "r"(Q[11]), "r"(Q[15]) : "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("bar.sync %0, %1;" :: "r"(g + 1), "r"(128) : "memory");
    if (tb == 0) {
      const long long e = (dof - dst_shift) >> 1;
      asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" :: "l"(&tdst), "r"((int)((e >> 0) & 63LL)), "r"((int)((e >> 6))), "r"(db) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    ++it;
    if (++s == 3) { s = 0; ph ^= 1u; }
  }
  if (tb == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
