// planner.hpp -- host planner: conversion quotient, tiling, thread mappings,
// optimal swizzle (paper Sec. 5.4 / Appendix), gather plans, plan cache.
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <string>
#include <vector>

#include "core.hpp"
#include "plan.hpp"

namespace ll {

// Result of the paper's optimal-swizzling construction (P:685-713,
// P:1104-1130) on a tile-local space of d bits.
struct SwizzleResult {
  std::vector<u64> vect, bank, idx;     // columns of S: offset bits -> tile-local vectors
  std::vector<u64> A_bank, B_bank, E, F, H, C;
  int v = 0, b = 0, ell = 0;
  bool unavoidable = false;
};

// A and B are given by their reg / lane / warp columns (tile-local vectors).
SwizzleResult optimal_swizzle(const std::vector<u64>& A_lane, const std::vector<u64>& B_lane,
                              const std::vector<u64>& V, int d, int elem_bytes);

// Lemma: wavefronts per instruction n * c, c from L_bank (A13).
int lemma_wavefronts(const SwizzleResult& s, const std::vector<u64>& lanes, int elem_bytes);

// Register-faithful warp-shuffle plan (LL_PATH_REGS_SHUFFLE): the paper's
// exchange on the layouts' own registers and lanes, for both
// directions (A -> B, and B -> A for loop-carried in-kernel timing).  Per
// round k of 2^|R|: every lane l sends word alpha_k ^ beta(l) (after the
// beta selects: T = R[. ^ beta(l)], send T[alpha_k]) to lane
// gamma_k ^ delta(l), which stores it at eps_k ^ zeta(l).  Executed by a
// kernel specialised for the plan at run time (NVRTC, jit.cpp): every
// register index is a compile-time constant, as in the paper's compiler.
struct ShuffleDir {
  std::vector<int> alpha, eps, gamma;      // per round k
  uint32_t beta[5] = {0}, zeta[5] = {0}, delta[5] = {0};
  uint32_t beta_any = 0, zeta_any = 0;
};
struct RegsShufflePlan {
  int nw = 0, nwords = 0;
  int64_t tile_bytes = 0, n_tiles = 0;
  std::vector<std::pair<int, int>> swaps;  // load-side element-bit swaps (A order -> B's words)
  ShuffleDir fwd, bwd;
};

struct ConvertPlan {
  int path = LL_PATH_GENERIC;
  int w = 0;
  int nA = 0, nB = 0;
  int64_t batch = 1;
  bool identity = false;
  bool padded = false;
  int op = 0;        // 0 = convert, 1 = fused mxfp4 upcast (NEXT #1)
  int64_t scale_row = 0;  // scales per row (K/32)
  int kb_bits = 0;        // bits of the packed-byte dim
  std::vector<u64> dst_cols;
  // smem path
  SmemPlan sp{};
  TmaDesc td{};      // LL_PATH_SMEM_TMA (source box)
  TmaDesc td_dst{};  // LL_PATH_SMEM_TMA_STORE (destination box)
  RegsPlan rp{};     // LL_PATH_REGS
  RegsShufflePlan rsp;  // LL_PATH_REGS_SHUFFLE
  int nv = 0, g = 0;
  int tile_bits = 0, r = 0, gw = 0;
  int pred_wf_ld = 0, pred_wf_st = 0;   // wavefronts per STS / LDS instruction
  // tile order: element positions of each outer (tile-index) bit in src / dst
  std::vector<int> tile_bit_src, tile_bit_dst;
  // shuffle path (warp tiles only)
  ShufflePlan shp{};
  ShuffleDir shd;     // the same exchange per round, for the NVRTC-specialised kernel
  bool shuffle_ok = false;
  int shuffle_rounds = 0;
  // broadcast dedup on the smem path:
  // the plan runs over virtual index spaces without the destination copy
  // bits and the unread source copy bits; src_phys / dst_phys map a virtual
  // bit to its buffer bit (empty: identity).  A virtual 16-byte vector spans
  // 2^ld_span / 2^st_span physical 16-byte vectors (copy bits inside it:
  // compacted / duplicated in registers), copy_off = byte offsets of the
  // destination copies above it (every destination vector stored at each).
  // Executed by the plan-compiled kernel only (jit_only; fallback: generic).
  std::vector<int> src_phys, dst_phys;
  int ld_span = 0, st_span = 0, ld_chunks = 1;
  int r_cap = 0;   // cap on the thread's register bits in plan_smem (0: none)
  // register permutation (LL_PATH_REGPERM): chunks of 2^rp_bits elements,
  // destination element e of a chunk = source element rp_src[e]
  int rp_bits = 0;
  std::vector<int> rp_src;
  std::vector<uint32_t> copy_off;
  bool jit_only = false;
  // generic path
  GenericPlan gp{};
  std::string json;
};

// Gather plan.  out[h] = src[h ^ Y(a(h) ^ idx[h])]: a(h) = the
// axis coordinate of L(h) (XOR of acol over h's bits), Y = the buffer vectors
// of the axis bits (L^{-1} e_axis_k).  Every Y lies in the low unit_bits
// buffer bits, so a gather never leaves an aligned unit of 2^unit_bits
// elements.  Paths:
//   LL_PATH_SHUFFLE  the unit fits one warp's registers (free mapping: lane l
//                    holds 16-byte vectors l, l + 32, ...): 2^|Y_reg| candidate
//                    shuffles per output (reading A19), compiled per plan;
//   LL_PATH_SMEM     the unit fits a CTA's shared memory: one bulk copy
//                    (cp.async.bulk) per unit, then LDS per output, compiled
//                    per plan (the paper's "legacy" gather);
//   LL_PATH_GENERIC  direct: source elements read through L1 (any layout).
struct GatherPlanHost {
  int path = LL_PATH_GENERIC;
  int w = 0;
  GatherPlan gp{};
  int n = 0, vb = 0;
  int unit_bits = 0;                // top buffer bit of span(Y) + 1
  int warp_bits = 0, cta_bits = 0;  // unit of the shuffle / smem kernel (>= unit_bits)
  int64_t batch = 1;
  std::vector<u64> Y;               // per axis bit
  std::vector<uint32_t> acol;       // per buffer bit
  bool shuffle_ok = false, smem_ok = false;
  bool paper_criterion = false;     // L_warp^axis = L_block^axis = 0 by the labels (A20)
  std::string json;
};

// gather.cpp
std::shared_ptr<GatherPlanHost> build_gather_plan(const Layout& L, int axis, int w, int path_req,
                                                  int64_t batch);
std::string gather_shfl_source(const GatherPlanHost& P, int timed);
std::string gather_smem_source(const GatherPlanHost& P, int timed);
cudaError_t launch_gather_jit(const GatherPlanHost& P, const void* src, const int32_t* idx,
                              void* out, int* err_flag, int max_ctas, cudaStream_t st,
                              std::string* err, int reps = 0, long long* cycles = nullptr);

// Shard `shard` of `n_shards` (a power of two) of a smem / shuffle / copy
// plan: the top log2(n_shards) bits of the src and dst indices must be the
// last tile-index bits and mapped identically (so every shard is one
// contiguous slice of each buffer).  Throws LL_ERR_UNSUPPORTED otherwise.
TileRange shard_range(const ConvertPlan& P, int n_shards, int shard);
// A shard that is a contiguous slice of one buffer and a pitched (2-D)
// region of the other: the top log2(n_shards) tile bits are the top index
// bits of side *side (0 = src, 1 = dst) and the contiguous run of index bits
// [*r0, *r0 + log2(n_shards)) of the other side.  The contiguous side's
// shift is its slice offset; the pitched side is addressed in place (shift 0).
TileRange shard_range_2d(const ConvertPlan& P, int n_shards, int shard, int* side, int* r0);

int planner_knob(const char* name, int dflt);
int planner_knob_version();
bool set_planner_knob(const std::string& name, int value);

// path_req: ll_path value (AUTO lets the planner choose).  Throws ll::Error.
std::shared_ptr<const ConvertPlan> get_convert_plan(const Layout& A, const Layout& B, int w,
                                                    int path_req, int64_t batch, int op = 0);
// jit.cpp: the NVRTC-specialised register-faithful shuffle kernel
std::string regs_shuffle_kernel_source(const RegsShufflePlan& p, int w);
cudaError_t launch_shuffle_jit(const ConvertPlan& P, const void* src, void* dst, int max_ctas,
                               cudaStream_t st, const TileRange& rg, std::string* err);
std::string shuffle_hbm_kernel_source(const ConvertPlan& P);
std::string smem_hbm_kernel_source(const ConvertPlan& P);
std::string upcast_hbm_kernel_source(const ConvertPlan& P);
cudaError_t launch_upcast_jit(const ConvertPlan& P, const void* src, void* dst,
                              const uint8_t* scales, int max_ctas, cudaStream_t st,
                              const TileRange& rg, std::string* err);
std::string regperm_kernel_source(const ConvertPlan& P);
cudaError_t launch_regperm_jit(const ConvertPlan& P, const void* src, void* dst, int max_ctas,
                               cudaStream_t st, const TileRange& rg, std::string* err);
cudaError_t launch_smem_jit(const ConvertPlan& P, const void* src, void* dst, int max_ctas,
                            cudaStream_t st, const TileRange& rg, std::string* err);
// the warp-specialised TMA kernels compiled per plan (LL_PATH_SMEM_TMA[_STORE])
std::string tma_hbm_kernel_source(const ConvertPlan& P, bool tma_store);
cudaError_t launch_tma_jit(const ConvertPlan& P, bool tma_store, const void* src, void* dst, int max_ctas,
                           cudaStream_t st, const TileRange& rg, std::string* err);
bool nvrtc_compile_check(const std::string& src, std::string* log, size_t* cubin_bytes);
cudaError_t launch_regs_shuffle(const RegsShufflePlan& p, int w, const void* src, void* dst,
                                int max_ctas, int reps, long long* cycles, cudaStream_t st,
                                std::string* err);

// jit.cpp: compile (cached) / launch a generated kernel (driver API)
cudaError_t jit_kernel(const std::string& src, const char* name, void** fn, std::string* err);
long long jit_first_wave_ctas(void* fn, int block, int smem);
cudaError_t jit_launch(void* fn, unsigned grid, unsigned block, unsigned smem, cudaStream_t st,
                       void** args, std::string* err, bool pdl = false);

std::shared_ptr<const GatherPlanHost> get_gather_plan(const Layout& L, int axis, int w,
                                                      int path_req, int64_t batch);

}  // namespace ll
