// planner_internal.hpp -- helpers shared by the planner's translation units
// (planner.cpp: quotient, smem / shuffle / generic plans, cache, shards;
// planner_tma.cpp: cp.async / TMA plans; planner_regs.cpp: register-faithful
// plans).  Not part of the library's interface.
#pragma once

#include <array>
#include <sstream>
#include <string>
#include <vector>

#include "planner.hpp"

namespace ll {
namespace detail {

int ilog2i(int x);
std::string vec_json(const std::vector<u64>& v);
std::string u32_json(const uint32_t* v, int n);
std::string ivec_json(const std::vector<int>& v);

// The paper's warp-shuffle exchange between two warp-local
// thread layouts given by their word-level register vectors (Aw / Bw, word
// order) and lane vectors (Al5 / Bl5): V is the word, I, E, F (ascending),
// G = {e_i ^ f_i}, R completes span(I u G); round k sends
// R[alpha(k) ^ beta(l)] to lane gamma(k) ^ delta(l), which stores it at word
// eps(k) ^ zeta(l).  ok = false if the exchange is not expressible so.
struct ShuffleCore {
  bool ok = false;
  int rounds = 0;
  std::vector<u64> I, E, F, Gv, R, alpha, epsm;
  std::vector<std::array<int, 3>> pre, post;
  uint32_t beta[5] = {0}, zeta[5] = {0}, delta[5] = {0}, beta_any = 0, zeta_any = 0;
  std::vector<uint8_t> gamma;
};

ShuffleCore shuffle_core(const std::vector<u64>& Aw, const std::vector<u64>& Al5,
                         const std::vector<u64>& Bw, const std::vector<u64>& Bl5, int LB);

// planner_tma.cpp
bool plan_async(ConvertPlan& P, const std::vector<u64>& X, std::ostringstream& js);
bool plan_tma(ConvertPlan& P, const std::vector<u64>& X, std::ostringstream& js);
bool plan_tma_store(ConvertPlan& P, const std::vector<u64>& X, std::ostringstream& js);

// planner_regs.cpp
bool plan_regs(ConvertPlan& P, const Layout& A, const Layout& B, const std::vector<u64>& X,
               std::ostringstream& js);
bool plan_regs_shuffle(ConvertPlan& P, const Layout& A, const Layout& B,
                       const std::vector<u64>& X, std::ostringstream& js);

}  // namespace detail
}  // namespace ll
