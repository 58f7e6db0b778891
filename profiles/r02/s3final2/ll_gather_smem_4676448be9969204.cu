extern "C" __global__ void __launch_bounds__(256) ll_gather_smem(
    const unsigned char* __restrict__ src, const int* __restrict__ idx,
    unsigned char* __restrict__ out, long long n_units, int* err, int check) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int tid = threadIdx.x;
  const unsigned sb = (unsigned)__cvta_generic_to_shared(smem);
  const unsigned bar0 = sb + 16384u;
  unsigned a_tid = 0;
  if (tid & 1) a_tid ^= 4u;
  if (tid & 2) a_tid ^= 8u;
  if (tid & 4) a_tid ^= 16u;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(bar0) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(bar0 + 8u) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](long long t, int s) {
    const unsigned bar = bar0 + 8u * s, st = sb + 8192u * s;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bar), "r"(8192u) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" :: "r"(st), "l"(src + (t << 10) * 4), "r"(4096u), "r"(bar) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" :: "r"(st + 4096u), "l"(idx + (t << 10)), "r"(4096u), "r"(bar) : "memory");
  };
  const long long g0 = blockIdx.x, gs = gridDim.x;
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  if (tid == 0) { if (g0 < n_units) issue(g0, 0); if (g0 + gs < n_units) issue(g0 + gs, 1); }
  int k = 0;
  for (long long t = g0; t < n_units; t += gs, ++k) {
    const int s = k & 1;
    const unsigned ph = (unsigned)(k >> 1) & 1u;
    asm volatile("{\n.reg .pred p;\nLL_GW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra LL_GW_%=;\n}\n" :: "r"(bar0 + 8u * s), "r"(ph) : "memory");
    const unsigned su = sb + 8192u * s, si = su + 4096u;
    const long long base = t << 10;
    unsigned a_unit = 0; { const long long r_ = t & 16383LL;
    }
    int I[1][4];
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(I[0][0]), "=r"(I[0][1]), "=r"(I[0][2]), "=r"(I[0][3]) : "r"(si + ((((unsigned)tid + 0u) << 2) + 0u) * 4u));
    { unsigned O[4] = {0, 0, 0, 0};
      { int ix = I[0][0];
        if (check && (unsigned)ix > 31u) atomicExch(err, 1);
        const unsigned d = (a_unit ^ a_tid ^ 0u ^ (unsigned)ix) & 31u;
        const unsigned hl = 0u | ((unsigned)tid << 2);
        const unsigned hs = (hl ^ (d << 0));
        unsigned v; asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(su + hs * 4u));
        O[0] = v; }
      { int ix = I[0][1];
        if (check && (unsigned)ix > 31u) atomicExch(err, 1);
        const unsigned d = (a_unit ^ a_tid ^ 1u ^ (unsigned)ix) & 31u;
        const unsigned hl = 1u | ((unsigned)tid << 2);
        const unsigned hs = (hl ^ (d << 0));
        unsigned v; asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(su + hs * 4u));
        O[1] = v; }
      { int ix = I[0][2];
        if (check && (unsigned)ix > 31u) atomicExch(err, 1);
        const unsigned d = (a_unit ^ a_tid ^ 2u ^ (unsigned)ix) & 31u;
        const unsigned hl = 2u | ((unsigned)tid << 2);
        const unsigned hs = (hl ^ (d << 0));
        unsigned v; asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(su + hs * 4u));
        O[2] = v; }
      { int ix = I[0][3];
        if (check && (unsigned)ix > 31u) atomicExch(err, 1);
        const unsigned d = (a_unit ^ a_tid ^ 3u ^ (unsigned)ix) & 31u;
        const unsigned hl = 3u | ((unsigned)tid << 2);
        const unsigned hs = (hl ^ (d << 0));
        unsigned v; asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(su + hs * 4u));
        O[3] = v; }
      asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(out + (base + (((long long)tid + 0) << 2)) * 4), "r"(O[0]), "r"(O[1]), "r"(O[2]), "r"(O[3]) : "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();   // every thread is done with stage s
    if (tid == 0 && t + 2 * gs < n_units) issue(t + 2 * gs, s);
  }
}
