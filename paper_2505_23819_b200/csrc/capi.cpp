// capi.cpp -- the extern "C" boundary of libll_b200.so (include/ll.h).
//
// Every entry point converts internal ll::Error / std::bad_alloc into an
// ll_status and a thread-local message; nothing throws across the ABI.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdlib>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <set>
#include <string>

#include "core.hpp"
#include "kernels.hpp"
#include "planner.hpp"

struct ll_layout_s {
  ll::Layout L;
};

namespace {

thread_local std::string g_err;
std::atomic<int64_t> g_launches{0};

ll_status fail(ll_status s, const std::string& m) {
  g_err = m;
  return s;
}

template <class F>
ll_status guarded(F&& f) {
  try {
    g_err.clear();
    return f();
  } catch (const ll::Error& e) {
    return fail(e.code, e.what());
  } catch (const std::bad_alloc&) {
    return fail(LL_ERR_OOM, "host allocation failed");
  } catch (const std::exception& e) {
    return fail(LL_ERR_ARG, e.what());
  }
}

ll_status cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return LL_OK;
  return fail(LL_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

int elem_bytes(int elem_bits) {
  switch (elem_bits) {
    case 8: return 1;
    case 16: return 2;
    case 32: return 4;
    case 64: return 8;
  }
  throw ll::Error(LL_ERR_ARG, "elem_bits must be 8, 16, 32 or 64 (got " + std::to_string(elem_bits) + ")");
}

ll_layout wrap(ll::Layout&& L) {
  auto* p = new ll_layout_s;
  p->L = std::move(L);
  return p;
}

void check_layout(ll_layout l, const char* what) {
  if (!l) throw ll::Error(LL_ERR_ARG, std::string(what) + ": NULL layout");
}

}  // namespace

extern "C" {

const char* ll_last_error(void) { return g_err.c_str(); }
const char* ll_version(void) { return "ll_b200 0.1 (sm_100a)"; }
int64_t ll_launch_count(void) { return g_launches.load(); }

ll_status ll_tune(const char* name, int value) {
  if (name && ll::set_planner_knob(name, value)) return LL_OK;
  if (ll::set_knob(name, value) != 0)
    return fail(LL_ERR_ARG, std::string("ll_tune: unknown knob '") + (name ? name : "") + "'");
  return LL_OK;
}

ll_status ll_layout_create(int n_in, const char* const* in_names, const int* in_bits, int n_out,
                           const char* const* out_names, const int* out_bits,
                           const int64_t* bases, ll_layout* out) {
  return guarded([&]() -> ll_status {
    if (!out) return fail(LL_ERR_ARG, "ll_layout_create: out is NULL");
    *out = nullptr;
    if (n_in < 0 || n_out < 0 || n_in > 16 || n_out > 16)
      return fail(LL_ERR_ARG, "ll_layout_create: n_in / n_out out of range [0, 16]");
    if ((n_in && (!in_names || !in_bits)) || (n_out && (!out_names || !out_bits)))
      return fail(LL_ERR_ARG, "ll_layout_create: NULL name or size array");
    ll::Layout L;
    std::set<std::string> seen;
    int tin = 0, tout = 0;
    for (int i = 0; i < n_in; ++i) {
      if (!in_names[i] || in_bits[i] < 0 || in_bits[i] > 62)
        return fail(LL_ERR_ARG, "ll_layout_create: bad input dim (bits must be in [0, 62])");
      if (!seen.insert(in_names[i]).second)
        return fail(LL_ERR_ARG, std::string("ll_layout_create: duplicate input dim '") + in_names[i] + "'");
      L.in.push_back({in_names[i], in_bits[i]});
      tin += in_bits[i];
    }
    seen.clear();
    for (int i = 0; i < n_out; ++i) {
      if (!out_names[i] || out_bits[i] < 0 || out_bits[i] > 62)
        return fail(LL_ERR_ARG, "ll_layout_create: bad output dim (bits must be in [0, 62])");
      if (!seen.insert(out_names[i]).second)
        return fail(LL_ERR_ARG, std::string("ll_layout_create: duplicate output dim '") + out_names[i] + "'");
      L.out.push_back({out_names[i], out_bits[i]});
      tout += out_bits[i];
    }
    if (tin > 62 || tout > 62) return fail(LL_ERR_ARG, "ll_layout_create: more than 62 bits");
    if (tin && !bases) return fail(LL_ERR_ARG, "ll_layout_create: bases is NULL");
    std::vector<int64_t> coords(n_out);
    for (int k = 0; k < tin; ++k) {
      for (int d = 0; d < n_out; ++d) {
        int64_t c = bases[(size_t)k * n_out + d];
        if (c < 0 || (out_bits[d] < 63 && c >= (int64_t(1) << out_bits[d])))
          return fail(LL_ERR_RANGE, "ll_layout_create: basis " + std::to_string(k) +
                                        " coordinate " + std::to_string(d) + " out of range");
        coords[d] = c;
      }
      L.cols.push_back(L.flatten(coords));
    }
    *out = wrap(std::move(L));
    return LL_OK;
  });
}

ll_status ll_layout_destroy(ll_layout l) {
  delete l;
  return LL_OK;
}

ll_status ll_layout_info(ll_layout l, int* n_in, int* n_out, int* in_bits_total,
                         int* out_bits_total) {
  return guarded([&]() -> ll_status {
    check_layout(l, "ll_layout_info");
    if (n_in) *n_in = (int)l->L.in.size();
    if (n_out) *n_out = (int)l->L.out.size();
    if (in_bits_total) *in_bits_total = l->L.in_bits();
    if (out_bits_total) *out_bits_total = l->L.out_bits();
    return LL_OK;
  });
}

ll_status ll_layout_get(ll_layout l, char (*in_names)[32], int* in_bits, char (*out_names)[32],
                        int* out_bits, int64_t* bases, size_t cap) {
  return guarded([&]() -> ll_status {
    check_layout(l, "ll_layout_get");
    const auto& L = l->L;
    for (size_t i = 0; i < L.in.size(); ++i) {
      if (in_names) { std::strncpy(in_names[i], L.in[i].name.c_str(), 31); in_names[i][31] = 0; }
      if (in_bits) in_bits[i] = L.in[i].bits;
    }
    for (size_t i = 0; i < L.out.size(); ++i) {
      if (out_names) { std::strncpy(out_names[i], L.out[i].name.c_str(), 31); out_names[i][31] = 0; }
      if (out_bits) out_bits[i] = L.out[i].bits;
    }
    if (bases) {
      if (cap < L.cols.size() * L.out.size()) return fail(LL_ERR_ARG, "ll_layout_get: bases too small");
      for (size_t k = 0; k < L.cols.size(); ++k) {
        auto c = L.unflatten(L.cols[k]);
        for (size_t d = 0; d < L.out.size(); ++d) bases[k * L.out.size() + d] = c[d];
      }
    }
    return LL_OK;
  });
}

ll_status ll_compose(ll_layout outer, ll_layout inner, ll_layout* out) {
  return guarded([&]() -> ll_status {
    check_layout(outer, "ll_compose");
    check_layout(inner, "ll_compose");
    if (!out) return fail(LL_ERR_ARG, "ll_compose: out is NULL");
    *out = wrap(ll::compose(outer->L, inner->L));
    return LL_OK;
  });
}

ll_status ll_invert(ll_layout l, ll_layout* out) {
  return guarded([&]() -> ll_status {
    check_layout(l, "ll_invert");
    if (!out) return fail(LL_ERR_ARG, "ll_invert: out is NULL");
    *out = wrap(ll::right_inverse(l->L));
    return LL_OK;
  });
}

ll_status ll_product(ll_layout a, ll_layout b, ll_layout* out) {
  return guarded([&]() -> ll_status {
    check_layout(a, "ll_product");
    check_layout(b, "ll_product");
    if (!out) return fail(LL_ERR_ARG, "ll_product: out is NULL");
    *out = wrap(ll::product(a->L, b->L));
    return LL_OK;
  });
}

ll_status ll_left_divide(ll_layout m, ll_layout m1, ll_layout* out) {
  return guarded([&]() -> ll_status {
    check_layout(m, "ll_left_divide");
    check_layout(m1, "ll_left_divide");
    if (!out) return fail(LL_ERR_ARG, "ll_left_divide: out is NULL");
    *out = wrap(ll::left_divide(m->L, m1->L));
    return LL_OK;
  });
}

ll_status ll_transpose(ll_layout l, const int* perm, ll_layout* out) {
  return guarded([&]() -> ll_status {
    check_layout(l, "ll_transpose");
    if (!out || (!perm && !l->L.out.empty())) return fail(LL_ERR_ARG, "ll_transpose: NULL argument");
    std::vector<int> p(perm, perm + l->L.out.size());
    *out = wrap(ll::shape_transpose(l->L, p));
    return LL_OK;
  });
}

ll_status ll_reshape(ll_layout l, int n_out, const char* const* out_names, const int* out_bits,
                     ll_layout* out) {
  return guarded([&]() -> ll_status {
    check_layout(l, "ll_reshape");
    if (!out || n_out < 0 || n_out > 16 || (n_out && (!out_names || !out_bits)))
      return fail(LL_ERR_ARG, "ll_reshape: bad arguments");
    std::vector<ll::Dim> d;
    std::set<std::string> seen;
    for (int i = 0; i < n_out; ++i) {
      if (!out_names[i] || !seen.insert(out_names[i]).second)
        return fail(LL_ERR_ARG, "ll_reshape: NULL or duplicate dim name");
      d.push_back({out_names[i], out_bits[i]});
    }
    *out = wrap(ll::shape_reshape(l->L, d));
    return LL_OK;
  });
}

ll_status ll_expand_dims(ll_layout l, int axis, const char* name, ll_layout* out) {
  return guarded([&]() -> ll_status {
    check_layout(l, "ll_expand_dims");
    if (!out || !name) return fail(LL_ERR_ARG, "ll_expand_dims: NULL argument");
    *out = wrap(ll::shape_expand_dims(l->L, axis, name));
    return LL_OK;
  });
}

ll_status ll_slice(ll_layout l, int axis, ll_layout* out) {
  return guarded([&]() -> ll_status {
    check_layout(l, "ll_slice");
    if (!out) return fail(LL_ERR_ARG, "ll_slice: NULL argument");
    *out = wrap(ll::shape_slice(l->L, axis));
    return LL_OK;
  });
}

ll_status ll_blocked(int rank, const int* shape_bits, const int* R, const int* T, const int* W,
                     const int* order, ll_layout* out) {
  return guarded([&]() -> ll_status {
    if (!out || rank <= 0 || rank > 16 || !shape_bits || !R || !T || !W || !order)
      return fail(LL_ERR_ARG, "ll_blocked: bad argument");
    auto v = [&](const int* a) { return std::vector<int>(a, a + rank); };
    *out = wrap(ll::make_blocked(v(shape_bits), v(R), v(T), v(W), v(order)));
    return LL_OK;
  });
}

ll_status ll_mma_tile(int operand, int bitwidth, ll_layout* out) {
  return guarded([&]() -> ll_status {
    if (!out) return fail(LL_ERR_ARG, "ll_mma_tile: NULL argument");
    *out = wrap(ll::make_mma_tile(operand, bitwidth));
    return LL_OK;
  });
}

ll_status ll_broadcast(ll_layout l, int axis, int bits, ll_layout* out) {
  return guarded([&]() -> ll_status {
    check_layout(l, "ll_broadcast");
    if (!out) return fail(LL_ERR_ARG, "ll_broadcast: NULL argument");
    *out = wrap(ll::shape_broadcast(l->L, axis, bits));
    return LL_OK;
  });
}

ll_status ll_join(ll_layout l, const char* name, ll_layout* out) {
  return guarded([&]() -> ll_status {
    check_layout(l, "ll_join");
    if (!out || !name) return fail(LL_ERR_ARG, "ll_join: NULL argument");
    *out = wrap(ll::shape_join(l->L, name));
    return LL_OK;
  });
}

ll_status ll_split(ll_layout l, ll_layout* out) {
  return guarded([&]() -> ll_status {
    check_layout(l, "ll_split");
    if (!out) return fail(LL_ERR_ARG, "ll_split: NULL argument");
    *out = wrap(ll::shape_split(l->L));
    return LL_OK;
  });
}

ll_status ll_apply(ll_layout l, const int64_t* in_coords, int64_t* out_coords) {
  return guarded([&]() -> ll_status {
    check_layout(l, "ll_apply");
    const auto& L = l->L;
    if ((!in_coords && !L.in.empty()) || (!out_coords && !L.out.empty()))
      return fail(LL_ERR_ARG, "ll_apply: NULL coordinates");
    ll::u64 h = 0;
    int off = 0;
    for (size_t i = 0; i < L.in.size(); ++i) {
      int64_t c = in_coords[i];
      if (c < 0 || c >= (int64_t(1) << L.in[i].bits))
        return fail(LL_ERR_RANGE, "ll_apply: coordinate of '" + L.in[i].name + "' out of range");
      h |= ll::u64(c) << off;
      off += L.in[i].bits;
    }
    auto o = L.unflatten(ll::f2_apply(L.cols, h));
    for (size_t d = 0; d < L.out.size(); ++d) out_coords[d] = o[d];
    return LL_OK;
  });
}

ll_status ll_layout_props(ll_layout l, int* surjective, int* distributed, int* memory) {
  return guarded([&]() -> ll_status {
    check_layout(l, "ll_layout_props");
    if (surjective) *surjective = l->L.surjective();
    if (distributed) *distributed = l->L.distributed();
    if (memory) *memory = l->L.memory();
    return LL_OK;
  });
}

ll_status ll_plan_describe(ll_layout src_layout, ll_layout dst_layout, int elem_bits, int path,
                           char* json, size_t cap, size_t* needed) {
  return guarded([&]() -> ll_status {
    check_layout(src_layout, "ll_plan_describe");
    check_layout(dst_layout, "ll_plan_describe");
    auto P = ll::get_convert_plan(src_layout->L, dst_layout->L, elem_bytes(elem_bits), path, 1);
    if (needed) *needed = P->json.size() + 1;
    if (json && cap) {
      std::strncpy(json, P->json.c_str(), cap - 1);
      json[cap - 1] = 0;
    }
    return LL_OK;
  });
}

ll_status ll_gather_describe(ll_layout layout, int axis, int elem_bits, int path, char* json,
                             size_t cap, size_t* needed) {
  return guarded([&]() -> ll_status {
    check_layout(layout, "ll_gather_describe");
    auto P = ll::get_gather_plan(layout->L, axis, elem_bytes(elem_bits), path, 1);
    if (needed) *needed = P->json.size() + 1;
    if (json && cap) {
      std::strncpy(json, P->json.c_str(), cap - 1);
      json[cap - 1] = 0;
    }
    return LL_OK;
  });
}

namespace {
// Streams and events of ll_convert_host, created once per device and reused
// (stream / event creation costs tens of microseconds per call).
struct HostPipe {
  static constexpr int kSlots = 4;
  std::mutex mu;
  cudaStream_t h2d = nullptr, comp = nullptr, d2h = nullptr;
  cudaEvent_t start, fin[3], ev_h2d[kSlots], ev_comp[kSlots], ev_d2h[kSlots];
};

HostPipe& host_pipe() {
  static std::mutex m;
  static HostPipe* pipes[64] = {nullptr};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) throw ll::Error(LL_ERR_CUDA, "ll_convert_host: bad device");
  std::lock_guard<std::mutex> lk(m);
  if (!pipes[dev]) {
    HostPipe* p = new HostPipe();
    auto ev = [](cudaEvent_t* e) { cudaEventCreateWithFlags(e, cudaEventDisableTiming); };
    cudaStreamCreateWithFlags(&p->h2d, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&p->comp, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&p->d2h, cudaStreamNonBlocking);
    ev(&p->start);
    for (auto& e : p->fin) ev(&e);
    for (int i = 0; i < HostPipe::kSlots; ++i) {
      ev(&p->ev_h2d[i]);
      ev(&p->ev_comp[i]);
      ev(&p->ev_d2h[i]);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      delete p;
      throw ll::Error(LL_ERR_CUDA, std::string("ll_convert_host: ") + cudaGetErrorString(e));
    }
    pipes[dev] = p;
  }
  return *pipes[dev];
}
}  // namespace

namespace {
ll_status run_convert(const void* src, ll_layout src_layout, void* dst, ll_layout dst_layout,
                      int elem_bits, const ll_convert_options* opts, ll_stream stream,
                      int n_shards, int shard, const ll::TileRange* rg_in = nullptr) {
  check_layout(src_layout, "ll_convert");
  check_layout(dst_layout, "ll_convert");
  const int w = elem_bytes(elem_bits);
  const int path_req = opts ? opts->path : LL_PATH_AUTO;
  const int64_t batch = opts && opts->batch > 0 ? opts->batch : 1;
  const int max_ctas = opts ? opts->max_ctas : 0;
  if (!src || !dst) return fail(LL_ERR_ARG, "ll_convert: NULL buffer");
  if ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15)
    return fail(LL_ERR_ARG, "ll_convert: buffers must be 16-byte aligned");
  auto P = ll::get_convert_plan(src_layout->L, dst_layout->L, w, path_req, batch);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  ll::TileRange rg{0, 0, 0, 0};
  if (rg_in) {
    rg = *rg_in;
  } else if (n_shards > 1) {
    rg = ll::shard_range(*P, n_shards, shard);
  } else if (P->path == LL_PATH_SMEM || P->path == LL_PATH_SMEM_NOSWIZZLE ||
             P->path == LL_PATH_SMEM_ASYNC || P->path == LL_PATH_SMEM_PADDED ||
             P->path == LL_PATH_SMEM_TMA || P->path == LL_PATH_SMEM_TMA_STORE) {
    rg.t1 = P->sp.tile.n_tiles;
  } else if (P->path == LL_PATH_SHUFFLE) {
    rg.t1 = P->shp.tile.n_tiles;
  }
  const size_t dst_bytes = (size_t)w << P->nB;
  switch (P->path) {
    case LL_PATH_REGPERM: {
      if (!rg_in && n_shards <= 1) {
        rg.t0 = 0;
        rg.t1 = ((int64_t(1) << P->nB) >> P->rp_bits) * batch;
      }
      ++g_launches;
      std::string err;
      cudaError_t e = ll::launch_regperm_jit(*P, src, dst, max_ctas, st, rg, &err);
      if (e != cudaSuccess && err != "cuLaunchKernel failed") {
        // compile / module problem, nothing launched: element-wise pull
        if (n_shards > 1) return fail(LL_ERR_UNSUPPORTED, "ll_convert_shard: regperm kernel unavailable: " + err);
        ll::GenericPlan gp = P->gp;
        return cuda_status(ll::launch_convert_generic(gp, w, src, dst, max_ctas, st),
                           "ll_convert (generic kernel, regperm fallback)");
      }
      if (e != cudaSuccess) return fail(LL_ERR_CUDA, "ll_convert (regperm): " + err);
      return LL_OK;
    }
    case LL_PATH_COPY: {
      ++g_launches;
      const size_t bytes = n_shards > 1 ? dst_bytes / n_shards : dst_bytes * batch;
      return cuda_status(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, st),
                         "ll_convert (copy)");
    }
    case LL_PATH_SHUFFLE:
      ++g_launches;
      if (ll::planner_knob("shuffle_jit", 1) && w <= 4) {
        // the plan compiled into its own kernel (NVRTC, constant register indices)
        std::string err;
        cudaError_t e = ll::launch_shuffle_jit(*P, src, dst, max_ctas, st, rg, &err);
        // NVRTC / module problems (nothing was launched): the generic shuffle kernel
        if (e != cudaSuccess && !err.empty() && err.rfind("cuLaunchKernel", 0) != 0) {
          return cuda_status(ll::launch_convert_shuffle(P->shp, w, P->nv, src, dst, max_ctas, st, rg),
                             "ll_convert (shuffle kernel)");
        }
        if (e != cudaSuccess && !err.empty()) return fail(LL_ERR_CUDA, "ll_convert (shuffle): " + err);
        return cuda_status(e, "ll_convert (specialised shuffle kernel)");
      }
      return cuda_status(ll::launch_convert_shuffle(P->shp, w, P->nv, src, dst, max_ctas, st, rg),
                         "ll_convert (shuffle kernel)");
    case LL_PATH_SMEM_ASYNC:
      ++g_launches;
      return cuda_status(ll::launch_convert_async(P->sp, w, P->nv, src, dst, max_ctas, st, rg),
                         "ll_convert (async smem kernel)");
    case LL_PATH_REGS_SHUFFLE: {
      if (n_shards > 1) return fail(LL_ERR_UNSUPPORTED, "ll_convert_shard: the regs_shuffle path is not shardable");
      ++g_launches;
      std::string err;
      cudaError_t e = ll::launch_regs_shuffle(P->rsp, w, src, dst, max_ctas, 1, nullptr, st, &err);
      if (e != cudaSuccess && !err.empty()) return fail(LL_ERR_CUDA, "ll_convert (regs_shuffle): " + err);
      return cuda_status(e, "ll_convert (register-faithful shuffle kernel)");
    }
    case LL_PATH_REGS:
      if (n_shards > 1) return fail(LL_ERR_UNSUPPORTED, "ll_convert_shard: the regs path is not shardable");
      ++g_launches;
      return cuda_status(ll::launch_convert_regs(P->rp, w, src, dst, max_ctas, 1, nullptr, st),
                         "ll_convert (register-faithful kernel)");
    case LL_PATH_SMEM_TMA_STORE:
    case LL_PATH_SMEM_TMA:
      ++g_launches;
      if (ll::planner_knob("tma_jit", 1)) {
        // warp-specialised TMA kernel compiled for the plan (NVRTC)
        std::string err;
        cudaError_t e = ll::launch_tma_jit(*P, P->path == LL_PATH_SMEM_TMA_STORE, src, dst, max_ctas, st, rg, &err);
        if (e == cudaSuccess || err.rfind("cuLaunchKernel", 0) == 0)
          return cuda_status(e, "ll_convert (specialised TMA kernel)");
        // compile / module / shape problem, nothing launched: the template kernels below
      }
      if (P->path == LL_PATH_SMEM_TMA)
        return cuda_status(ll::launch_convert_tma(P->sp, P->td, w, P->nv, src, dst, max_ctas, st, rg),
                           "ll_convert (TMA smem kernel)");
      return cuda_status(ll::launch_convert_tma_store(P->sp, P->td, P->td_dst, w, P->nv, src, dst,
                                                      max_ctas, st, rg),
                         "ll_convert (TMA load/store kernel)");
    case LL_PATH_SMEM:
      if (ll::planner_knob("smem_jit", 1) && !P->sp.pad) {
        ++g_launches;
        std::string err;
        cudaError_t e = ll::launch_smem_jit(*P, src, dst, max_ctas, st, rg, &err);
        if (e == cudaSuccess || err.rfind("cuLaunchKernel", 0) == 0)
          return cuda_status(e, "ll_convert (specialised smem kernel)");
        // compile / module problem, nothing launched (a successful launch
        // returns cudaSuccess): the generic smem kernel below
        --g_launches;
      }
      if (P->jit_only) {
        // broadcast-dedup plans exist only as compiled kernels: element-wise pull
        if (n_shards > 1) return fail(LL_ERR_UNSUPPORTED, "ll_convert_shard: this plan needs the compiled smem kernel");
        ++g_launches;
        return cuda_status(ll::launch_convert_generic(P->gp, w, src, dst, max_ctas, st),
                           "ll_convert (generic kernel, broadcast plan)");
      }
      [[fallthrough]];
    case LL_PATH_SMEM_NOSWIZZLE:
    case LL_PATH_SMEM_PADDED:
      ++g_launches;
      return cuda_status(ll::launch_convert_smem(P->sp, w, P->nv, P->g, src, dst, max_ctas, st, rg),
                         "ll_convert (smem kernel)");
    default:
      if (n_shards > 1) return fail(LL_ERR_UNSUPPORTED, "ll_convert_shard: generic plans are not shardable");
      ++g_launches;
      return cuda_status(ll::launch_convert_generic(P->gp, w, src, dst, max_ctas, st),
                         "ll_convert (generic kernel)");
  }
}
}  // namespace

ll_status ll_convert_ex(const void* src, ll_layout src_layout, void* dst, ll_layout dst_layout,
                        int elem_bits, const ll_convert_options* opts, ll_stream stream) {
  return guarded([&]() -> ll_status {
    return run_convert(src, src_layout, dst, dst_layout, elem_bits, opts, stream, 1, 0);
  });
}

ll_status ll_convert_inkernel_timed(const void* src, ll_layout src_layout, void* dst,
                                    ll_layout dst_layout, int elem_bits, int64_t batch, int path,
                                    int reps, long long* cycles, ll_stream stream) {
  return guarded([&]() -> ll_status {
    check_layout(src_layout, "ll_convert_inkernel_timed");
    check_layout(dst_layout, "ll_convert_inkernel_timed");
    const int w = elem_bytes(elem_bits);
    if (!src || !dst) return fail(LL_ERR_ARG, "ll_convert_inkernel_timed: NULL buffer");
    if ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15)
      return fail(LL_ERR_ARG, "ll_convert_inkernel_timed: buffers must be 16-byte aligned");
    if (reps < 1) return fail(LL_ERR_ARG, "ll_convert_inkernel_timed: reps < 1");
    if (path != LL_PATH_REGS && path != LL_PATH_REGS_SHUFFLE)
      return fail(LL_ERR_ARG, "ll_convert_inkernel_timed: path must be LL_PATH_REGS or LL_PATH_REGS_SHUFFLE");
    auto P = ll::get_convert_plan(src_layout->L, dst_layout->L, w, path, batch > 0 ? batch : 1);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    ++g_launches;
    if (P->path == LL_PATH_REGS)
      return cuda_status(ll::launch_convert_regs(P->rp, w, src, dst, 0, reps, cycles, st),
                         "ll_convert_inkernel_timed");
    std::string err;
    cudaError_t e = ll::launch_regs_shuffle(P->rsp, w, src, dst, 0, reps, cycles, st, &err);
    if (e != cudaSuccess && !err.empty()) return fail(LL_ERR_CUDA, "ll_convert_inkernel_timed: " + err);
    return cuda_status(e, "ll_convert_inkernel_timed");
  });
}

ll_status ll_jit_source(ll_layout src_layout, ll_layout dst_layout, int elem_bits, int compile,
                        char* buf, size_t cap, size_t* need) {
  return guarded([&]() -> ll_status {
    check_layout(src_layout, "ll_jit_source");
    check_layout(dst_layout, "ll_jit_source");
    const int w = elem_bytes(elem_bits);
    std::string out;
    if (compile & 96) {  // the compiled TMA kernels (32: LL_PATH_SMEM_TMA, 64: _TMA_STORE)
      const bool store = (compile & 64) != 0;
      auto P = ll::get_convert_plan(src_layout->L, dst_layout->L, w,
                                    store ? LL_PATH_SMEM_TMA_STORE : LL_PATH_SMEM_TMA, 1);
      out = ll::tma_hbm_kernel_source(*P, store);
      if (out.empty()) return fail(LL_ERR_UNSUPPORTED, "ll_jit_source: the TMA tile does not fit two stages");
    } else if (compile & 16) {  // the register-permutation kernel (LL_PATH_REGPERM)
      auto P = ll::get_convert_plan(src_layout->L, dst_layout->L, w, LL_PATH_REGPERM, 1);
      out = ll::regperm_kernel_source(*P);
    } else if (compile & 8) {  // the fused mxfp4 upcast kernel (src / dst = the config-5 byte layouts)
      auto P = ll::get_convert_plan(src_layout->L, dst_layout->L, 1, LL_PATH_AUTO, 1, 1);
      out = ll::upcast_hbm_kernel_source(*P);
    } else if (compile & 4) {  // the HBM shared-memory conversion kernel (LL_PATH_SMEM)
      auto P = ll::get_convert_plan(src_layout->L, dst_layout->L, w, LL_PATH_SMEM, 1);
      out = ll::smem_hbm_kernel_source(*P);
    } else if (compile & 2) {  // the HBM shuffle conversion kernel (LL_PATH_SHUFFLE)
      auto P = ll::get_convert_plan(src_layout->L, dst_layout->L, w, LL_PATH_SHUFFLE, 1);
      out = ll::shuffle_hbm_kernel_source(*P);
    } else {
      auto P = ll::get_convert_plan(src_layout->L, dst_layout->L, w, LL_PATH_REGS_SHUFFLE, 1);
      out = ll::regs_shuffle_kernel_source(P->rsp, w);
    }
    if (compile & 1) {
      std::string log;
      size_t cubin = 0;
      const bool ok = ll::nvrtc_compile_check(out, &log, &cubin);
      out = std::string("{\"compiled\":") + (ok ? "true" : "false") + ",\"cubin_bytes\":" +
            std::to_string(cubin) + "}";
      if (!ok) return fail(LL_ERR_UNSUPPORTED, "ll_jit_source: NVRTC failed: " + log.substr(0, 300));
    }
    if (need) *need = out.size() + 1;
    if (buf && cap) {
      const size_t n = std::min(cap - 1, out.size());
      std::memcpy(buf, out.data(), n);
      buf[n] = 0;
    }
    return LL_OK;
  });
}

ll_status ll_gather_jit_source(ll_layout layout, int axis, int elem_bits, int path, int mode,
                              char* buf, size_t cap, size_t* need) {
  return guarded([&]() -> ll_status {
    check_layout(layout, "ll_gather_jit_source");
    const int w = elem_bytes(elem_bits);
    if (path != LL_PATH_SHUFFLE && path != LL_PATH_SMEM)
      return fail(LL_ERR_ARG, "ll_gather_jit_source: path must be SHUFFLE or SMEM");
    auto P = ll::get_gather_plan(layout->L, axis, w, path, 1);
    const int timed = (mode & 2) ? 1 : 0;
    std::string out = path == LL_PATH_SHUFFLE ? ll::gather_shfl_source(*P, timed)
                                              : ll::gather_smem_source(*P, timed);
    if (mode & 1) {
      std::string log;
      size_t cubin = 0;
      const bool ok = ll::nvrtc_compile_check(out, &log, &cubin);
      out = std::string("{\"compiled\":") + (ok ? "true" : "false") + ",\"cubin_bytes\":" +
            std::to_string(cubin) + "}";
      if (!ok) return fail(LL_ERR_UNSUPPORTED, "ll_gather_jit_source: NVRTC failed: " + log.substr(0, 600));
    }
    if (need) *need = out.size() + 1;
    if (buf && cap) {
      const size_t n = std::min(cap - 1, out.size());
      std::memcpy(buf, out.data(), n);
      buf[n] = 0;
    }
    return LL_OK;
  });
}

ll_status ll_gather_timed(const void* src, const int32_t* idx, void* out, ll_layout layout,
                          int axis, int elem_bits, int path, int reps, long long* cycles,
                          ll_stream stream) {
  return guarded([&]() -> ll_status {
    check_layout(layout, "ll_gather_timed");
    const int w = elem_bytes(elem_bits);
    if (!src || !idx || !out) return fail(LL_ERR_ARG, "ll_gather_timed: NULL buffer");
    if (reps < 1) return fail(LL_ERR_ARG, "ll_gather_timed: reps < 1");
    if (path != LL_PATH_SHUFFLE && path != LL_PATH_SMEM)
      return fail(LL_ERR_ARG, "ll_gather_timed: path must be SHUFFLE or SMEM");
    auto P = ll::get_gather_plan(layout->L, axis, w, path, 1);
    std::string err;
    ++g_launches;
    cudaError_t e = ll::launch_gather_jit(*P, src, idx, out, nullptr, 1,
                                          reinterpret_cast<cudaStream_t>(stream), &err, reps, cycles);
    if (e != cudaSuccess) return fail(LL_ERR_CUDA, "ll_gather_timed: " + (err.empty() ? std::string(cudaGetErrorString(e)) : err));
    return LL_OK;
  });
}

ll_status ll_convert_regs_timed(const void* src, ll_layout src_layout, void* dst,
                                ll_layout dst_layout, int elem_bits, int64_t batch, int reps,
                                long long* cycles, ll_stream stream) {
  return ll_convert_inkernel_timed(src, src_layout, dst, dst_layout, elem_bits, batch,
                                   LL_PATH_REGS, reps, cycles, stream);
}

ll_status ll_mxfp4_scale_layout(ll_layout dst_layout, ll_layout* out) {
  return guarded([&]() -> ll_status {
    check_layout(dst_layout, "ll_mxfp4_scale_layout");
    if (!out) return fail(LL_ERR_ARG, "ll_mxfp4_scale_layout: NULL argument");
    const ll::Layout& B = dst_layout->L;
    if (B.out.size() != 2 || B.out[1].bits < 4)
      return fail(LL_ERR_SHAPE, "ll_mxfp4_scale_layout: the layout must map to [m, kb] with >= 4 kb bits");
    // the projection (m, kb) -> (m, kb >> 4): one E8M0 scale per 16 packed
    // bytes (32 fp4 values) along K; kb bits 0-3 become zero columns
    const int kbb = B.out[1].bits;
    const ll::u64 kmask = (ll::u64(1) << kbb) - 1;
    ll::Layout S;
    S.in = B.in;
    S.out = {ll::Dim{B.out[0].name, B.out[0].bits}, ll::Dim{"g", kbb - 4}};
    for (ll::u64 c : B.cols) S.cols.push_back(((c >> kbb) << (kbb - 4)) | ((c & kmask) >> 4));
    *out = wrap(std::move(S));
    return LL_OK;
  });
}

ll_status ll_mxfp4_upcast(const void* packed, ll_layout src_layout, const uint8_t* scales,
                          void* dst_bf16, ll_layout dst_layout, const ll_convert_options* opts,
                          ll_stream stream) {
  return guarded([&]() -> ll_status {
    check_layout(src_layout, "ll_mxfp4_upcast");
    check_layout(dst_layout, "ll_mxfp4_upcast");
    if (!packed || !scales || !dst_bf16) return fail(LL_ERR_ARG, "ll_mxfp4_upcast: NULL buffer");
    if ((reinterpret_cast<uintptr_t>(packed) & 15) || (reinterpret_cast<uintptr_t>(dst_bf16) & 31))
      return fail(LL_ERR_ARG, "ll_mxfp4_upcast: packed must be 16-byte and dst_bf16 32-byte aligned");
    const int64_t batch = opts && opts->batch > 0 ? opts->batch : 1;
    if (batch != 1) return fail(LL_ERR_UNSUPPORTED, "ll_mxfp4_upcast: batch must be 1");
    auto P = ll::get_convert_plan(src_layout->L, dst_layout->L, 1, LL_PATH_AUTO, 1, 1);
    ll::TileRange rg{0, P->sp.tile.n_tiles, 0, 0};
    ++g_launches;
    if (ll::planner_knob("upcast_jit", 1) && P->sp.sc_nz <= 2) {
      std::string err;
      cudaError_t e = ll::launch_upcast_jit(*P, packed, dst_bf16, scales, opts ? opts->max_ctas : 0,
                                            reinterpret_cast<cudaStream_t>(stream), rg, &err);
      if (e == cudaSuccess || err.rfind("cuLaunchKernel", 0) == 0)
        return cuda_status(e, "ll_mxfp4_upcast (specialised kernel)");
      // compile / module problem, nothing launched: the template kernel below
    }
    return cuda_status(ll::launch_mxfp4_upcast(P->sp, P->nv, P->g, packed, dst_bf16, scales,
                                               opts ? opts->max_ctas : 0,
                                               reinterpret_cast<cudaStream_t>(stream), rg),
                       "ll_mxfp4_upcast");
  });
}

ll_status ll_checksum(const void* buf, int64_t n_elems, int elem_bits, int indexed,
                      int64_t index_base, uint64_t* result, ll_stream stream) {
  return guarded([&]() -> ll_status {
    const int w = elem_bytes(elem_bits);
    if (!buf || !result) return fail(LL_ERR_ARG, "ll_checksum: NULL pointer");
    if (n_elems < 0) return fail(LL_ERR_ARG, "ll_checksum: n_elems < 0");
    if (reinterpret_cast<uintptr_t>(buf) & 15)
      return fail(LL_ERR_ARG, "ll_checksum: buffer must be 16-byte aligned");
    ++g_launches;
    return cuda_status(ll::launch_checksum(buf, n_elems, w, indexed != 0, index_base,
                                           reinterpret_cast<unsigned long long*>(result),
                                           reinterpret_cast<cudaStream_t>(stream)),
                       "ll_checksum");
  });
}

ll_status ll_convert_shard(const void* src_slice, ll_layout src_layout, void* dst_slice,
                           ll_layout dst_layout, int elem_bits, int n_shards, int shard,
                           const ll_convert_options* opts, ll_stream stream) {
  return guarded([&]() -> ll_status {
    return run_convert(src_slice, src_layout, dst_slice, dst_layout, elem_bits, opts, stream,
                       n_shards, shard);
  });
}

ll_status ll_shard_describe(ll_layout src_layout, ll_layout dst_layout, int elem_bits, int path,
                            int n_shards, int shard, int64_t* out4) {
  return guarded([&]() -> ll_status {
    check_layout(src_layout, "ll_shard_describe");
    check_layout(dst_layout, "ll_shard_describe");
    if (!out4) return fail(LL_ERR_ARG, "ll_shard_describe: out is NULL");
    const int w = elem_bytes(elem_bits);
    auto P = ll::get_convert_plan(src_layout->L, dst_layout->L, w, path, 1);
    auto rg = ll::shard_range(*P, n_shards, shard);
    const int64_t sbytes = ((int64_t)w << P->nA) / n_shards, dbytes = ((int64_t)w << P->nB) / n_shards;
    out4[0] = rg.src_shift;
    out4[1] = rg.src_shift + sbytes;
    out4[2] = rg.dst_shift;
    out4[3] = rg.dst_shift + dbytes;
    return LL_OK;
  });
}

ll_status ll_shard_describe_2d(ll_layout src_layout, ll_layout dst_layout, int elem_bits, int path,
                               int n_shards, int shard, int64_t* out6) {
  return guarded([&]() -> ll_status {
    check_layout(src_layout, "ll_shard_describe_2d");
    check_layout(dst_layout, "ll_shard_describe_2d");
    if (!out6) return fail(LL_ERR_ARG, "ll_shard_describe_2d: out is NULL");
    const int w = elem_bytes(elem_bits);
    auto P = ll::get_convert_plan(src_layout->L, dst_layout->L, w, path, 1);
    int side = 0, r0 = 0;
    auto rg = ll::shard_range_2d(*P, n_shards, shard, &side, &r0);
    const int64_t slice = ((int64_t)w << (side == 0 ? P->nA : P->nB)) / n_shards;
    out6[0] = side;
    out6[1] = r0;
    out6[2] = side == 0 ? rg.src_shift : rg.dst_shift;
    out6[3] = out6[2] + slice;
    out6[4] = (int64_t)w << r0;
    out6[5] = ((int64_t)w << r0) * n_shards;
    return LL_OK;
  });
}

ll_status ll_convert(const void* src, ll_layout src_layout, void* dst, ll_layout dst_layout,
                     int elem_bits, ll_stream stream) {
  return ll_convert_ex(src, src_layout, dst, dst_layout, elem_bits, nullptr, stream);
}

ll_status ll_gather_ex(const void* src, const int32_t* idx, void* out, ll_layout layout, int axis,
                       int elem_bits, const ll_convert_options* opts, ll_stream stream) {
  return guarded([&]() -> ll_status {
    check_layout(layout, "ll_gather");
    const int w = elem_bytes(elem_bits);
    if (!src || !idx || !out) return fail(LL_ERR_ARG, "ll_gather: NULL buffer");
    if ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(idx) |
         reinterpret_cast<uintptr_t>(out)) & 15)
      return fail(LL_ERR_ARG, "ll_gather: buffers must be 16-byte aligned");
    const int path_req = opts ? opts->path : LL_PATH_AUTO;
    const int64_t batch = opts && opts->batch > 0 ? opts->batch : 1;
    const int max_ctas = opts ? opts->max_ctas : 0;
    auto P = ll::get_gather_plan(layout->L, axis, w, path_req, batch);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const char* chk = std::getenv("LL_GATHER_CHECK");
    const bool check = chk && chk[0] == '1';
    int* derr = nullptr;
    ll::GatherPlan gp = P->gp;
    if (check) {
      if (cudaMalloc(&derr, sizeof(int)) != cudaSuccess) return fail(LL_ERR_CUDA, "ll_gather: cudaMalloc");
      cudaMemsetAsync(derr, 0, sizeof(int), st);
      gp.check = 1;
    }
    ++g_launches;
    ll_status s = LL_OK;
    bool done = false;
    if (P->path == LL_PATH_SHUFFLE || P->path == LL_PATH_SMEM) {
      // compiled per plan (gather.cpp); a compile / module failure (nothing
      // launched) falls back to the direct kernel, which takes any layout
      ll::GatherPlanHost hp = *P;
      hp.gp.check = check ? 1 : 0;
      std::string err;
      cudaError_t e = ll::launch_gather_jit(hp, src, idx, out, derr, max_ctas, st, &err);
      if (e == cudaSuccess || err == "cuLaunchKernel failed") {
        s = e == cudaSuccess ? LL_OK : fail(LL_ERR_CUDA, "ll_gather (compiled kernel): " + err);
        done = true;
      }
    }
    if (!done)
      s = cuda_status(ll::launch_gather(gp, w, false, src, idx, out, derr, max_ctas, st),
                      "ll_gather");
    if (check) {
      int h = 0;
      cudaMemcpyAsync(&h, derr, sizeof(int), cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      cudaFree(derr);
      if (s == LL_OK && h) return fail(LL_ERR_RANGE, "ll_gather: index out of range");
    }
    return s;
  });
}

ll_status ll_gather(const void* src, const int32_t* idx, void* out, ll_layout layout, int axis,
                    int elem_bits, ll_stream stream) {
  return ll_gather_ex(src, idx, out, layout, axis, elem_bits, nullptr, stream);
}

ll_status ll_convert_host(const void* src_host, ll_layout src_layout, void* dst_host,
                          ll_layout dst_layout, int elem_bits, int64_t batch, void* dev_src,
                          void* dev_dst, size_t scratch_bytes, ll_stream stream) {
  return guarded([&]() -> ll_status {
    check_layout(src_layout, "ll_convert_host");
    check_layout(dst_layout, "ll_convert_host");
    const int w = elem_bytes(elem_bits);
    if (!src_host || !dst_host || !dev_src || !dev_dst)
      return fail(LL_ERR_ARG, "ll_convert_host: NULL buffer");
    if (batch < 1) batch = 1;
    const size_t sb = (size_t)w << src_layout->L.in_bits();
    const size_t db = (size_t)w << dst_layout->L.in_bits();
    const size_t unit = sb > db ? sb : db;
    // chunk target (knob host_chunk_mb; default by chunk kind, measured:
    // shards of one large instance 32 MiB -- config 5 92.8 vs 91.6 GB/s at
    // 16 --, whole batched instances 16 MiB -- config 2 85 vs 81 at 32)
    const int chunk_knob = ll::planner_knob("host_chunk_mb", 0);
    const size_t target_sh = (size_t)(chunk_knob > 0 ? chunk_knob : 32) << 20;
    const size_t target = (size_t)(chunk_knob > 0 ? chunk_knob : 16) << 20;
    const int max_slots = std::max(1, std::min(HostPipe::kSlots, ll::planner_knob("host_slots", 2)));
    // chunking: whole layout instances (batch elements), or -- for a single
    // large instance -- shards (contiguous slices of both buffers)
    // (a chunk must also fit one slot of the caller's scratch)
    const size_t cap = std::max<size_t>(1, std::min(target_sh, scratch_bytes));
    int n_sh = 1;
    if (batch == 1 && unit > cap) {
      auto P = ll::get_convert_plan(src_layout->L, dst_layout->L, w, LL_PATH_AUTO, 1);
      int want = 1;
      while ((unit / want) > cap && want < (1 << 12)) want *= 2;
      for (int ns = want; ns > 1; ns /= 2) {
        try {
          ll::shard_range(*P, ns, 0);
          n_sh = ns;
          break;
        } catch (const ll::Error&) {
        }
      }
    }
    // a single instance that cannot be cut into slices contiguous in both
    // buffers (a transpose): shards contiguous on one side and a pitched
    // region of >= 1 KiB rows on the other, the pitched side staged whole in
    // its scratch buffer and copied with cudaMemcpy2DAsync
    // (pitched shards keep the 16 MiB target: config 3 85 vs 79 GB/s at 32)
    const size_t cap2d = std::max<size_t>(1, std::min(target, scratch_bytes));
    if (batch == 1 && unit > cap2d && n_sh == 1 && ll::planner_knob("host_2d", 1)) {
      auto P = ll::get_convert_plan(src_layout->L, dst_layout->L, w, LL_PATH_AUTO, 1);
      int want = 2;
      while ((unit / want) > cap2d && want < (1 << 12)) want *= 2;
      for (int ns = want; ns > 1; ns /= 2) {
        int side = 0, r0 = 0;
        try {
          ll::shard_range_2d(*P, ns, 0, &side, &r0);
        } catch (const ll::Error&) {
          continue;
        }
        const size_t whole = side == 0 ? db : sb;   // the pitched side
        const size_t slice = (side == 0 ? sb : db) / ns;
        const size_t width = (size_t)w << r0;
        if (width < 1024 || scratch_bytes < whole || scratch_bytes < slice) continue;
        const size_t pitch = width * ns, height = whole / pitch;
        const int nslot = (int)std::max<size_t>(1, std::min<size_t>(max_slots, scratch_bytes / slice));
        HostPipe& hp = host_pipe();
        std::lock_guard<std::mutex> lk(hp.mu);
        cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
        cudaEventRecord(hp.start, st);
        cudaStreamWaitEvent(hp.h2d, hp.start, 0);
        cudaStreamWaitEvent(hp.comp, hp.start, 0);
        cudaStreamWaitEvent(hp.d2h, hp.start, 0);
        ll_status s = LL_OK;
        for (int i = 0; i < ns && s == LL_OK; ++i) {
          const int slot = i % nslot;
          const ll::TileRange rg = ll::shard_range_2d(*P, ns, i, &side, &r0);
          char* ds = (char*)dev_src + (side == 0 ? (size_t)slot * slice : 0);
          char* dd = (char*)dev_dst + (side == 0 ? 0 : (size_t)slot * slice);
          // the contiguous side's slot is reused every nslot chunks
          if (side == 0 && i >= nslot) cudaStreamWaitEvent(hp.h2d, hp.ev_comp[slot], 0);
          if (side == 0)
            cudaMemcpyAsync(ds, (const char*)src_host + i * slice, slice, cudaMemcpyHostToDevice, hp.h2d);
          else
            cudaMemcpy2DAsync(ds + i * width, pitch, (const char*)src_host + i * width, pitch, width,
                              height, cudaMemcpyHostToDevice, hp.h2d);
          cudaEventRecord(hp.ev_h2d[slot], hp.h2d);
          cudaStreamWaitEvent(hp.comp, hp.ev_h2d[slot], 0);
          if (side == 1 && i >= nslot) cudaStreamWaitEvent(hp.comp, hp.ev_d2h[slot], 0);
          ll_convert_options o{};
          o.path = LL_PATH_AUTO;
          s = guarded([&] {
            return run_convert(ds, src_layout, dd, dst_layout, elem_bits, &o, (ll_stream)hp.comp,
                               1, 0, &rg);
          });
          cudaEventRecord(hp.ev_comp[slot], hp.comp);
          cudaStreamWaitEvent(hp.d2h, hp.ev_comp[slot], 0);
          if (side == 0)
            cudaMemcpy2DAsync((char*)dst_host + i * width, pitch, dd + i * width, pitch, width, height,
                              cudaMemcpyDeviceToHost, hp.d2h);
          else
            cudaMemcpyAsync((char*)dst_host + i * slice, dd, slice, cudaMemcpyDeviceToHost, hp.d2h);
          cudaEventRecord(hp.ev_d2h[slot], hp.d2h);
        }
        cudaEventRecord(hp.fin[0], hp.h2d);
        cudaEventRecord(hp.fin[1], hp.comp);
        cudaEventRecord(hp.fin[2], hp.d2h);
        for (int k = 0; k < 3; ++k) cudaStreamWaitEvent(st, hp.fin[k], 0);
        cudaError_t e = cudaStreamSynchronize(st);
        if (s != LL_OK) return s;
        return cuda_status(e, "ll_convert_host");
      }
    }
    int64_t n_chunks, per_chunk = 1;
    size_t cs_src, cs_dst;  // bytes per chunk (src / dst side)
    if (n_sh > 1) {
      n_chunks = n_sh;
      cs_src = sb / n_sh;
      cs_dst = db / n_sh;
    } else {
      if (scratch_bytes < unit)
        return fail(LL_ERR_ARG, "ll_convert_host: scratch smaller than one layout instance");
      per_chunk = (int64_t)std::max<size_t>(1, target / unit);
      per_chunk = std::min<int64_t>(per_chunk, (int64_t)(scratch_bytes / unit));
      per_chunk = std::min<int64_t>(per_chunk, batch);
      n_chunks = (batch + per_chunk - 1) / per_chunk;
      cs_src = per_chunk * sb;
      cs_dst = per_chunk * db;
    }
    const size_t cs = cs_src > cs_dst ? cs_src : cs_dst;
    if (scratch_bytes < cs) return fail(LL_ERR_ARG, "ll_convert_host: scratch smaller than one chunk");
    const int nslot = (int)std::max<size_t>(1, std::min<size_t>(max_slots, scratch_bytes / cs));

    // Three streams: copy-in (H2D), compute, copy-out (D2H).  One stream per
    // direction keeps each copy engine working on one chunk at a time in
    // order (copies of one direction on several streams share the link and
    // finish later); per-slot events hand chunks down the pipeline and guard
    // slot reuse: H2D(i) waits for the kernel of chunk i-nslot (its source
    // slot), the kernel of chunk i waits for D2H(i-nslot) (its destination
    // slot).  The H2D of chunk i+1, the kernel of chunk i and the D2H of
    // chunk i-1 overlap.
    HostPipe& hp = host_pipe();
    std::lock_guard<std::mutex> lk(hp.mu);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    cudaEventRecord(hp.start, st);
    cudaStreamWaitEvent(hp.h2d, hp.start, 0);
    cudaStreamWaitEvent(hp.comp, hp.start, 0);
    cudaStreamWaitEvent(hp.d2h, hp.start, 0);
    // shard chunks: (n_shards, shard) per chunk.  Ramp (knob host_ramp = R
    // levels, default 0): the first and the last shard cut into pieces of
    // 1/2^R .. 1/2 of a chunk, so the pipeline would fill and drain on small
    // copies -- measured no faster on config 5 (92.6 vs 92.8 GB/s,
    // profiles/r02/s3o), kept as a knob
    std::vector<std::pair<int, int>> sched;
    if (n_sh > 1) {
      int R = std::max(0, std::min(4, ll::planner_knob("host_ramp", 0)));
      auto P = ll::get_convert_plan(src_layout->L, dst_layout->L, w, LL_PATH_AUTO, 1);
      while (R > 0 && n_sh >= 2) {
        try {
          ll::shard_range(*P, n_sh << R, 0);
          break;
        } catch (const ll::Error&) {
          --R;
        }
      }
      if (R > 0 && n_sh >= 2) {
        const int fin = n_sh << R;
        sched.push_back({fin, 0});
        for (int L = R; L >= 1; --L) sched.push_back({n_sh << L, 1});
        for (int k = 1; k + 1 < n_sh; ++k) sched.push_back({n_sh, k});
        for (int L = 1; L <= R; ++L) sched.push_back({n_sh << L, (n_sh << L) - 2});
        sched.push_back({fin, fin - 1});
      } else {
        for (int k = 0; k < n_sh; ++k) sched.push_back({n_sh, k});
      }
      n_chunks = (int64_t)sched.size();
    }
    ll_status s = LL_OK;
    for (int64_t i = 0; i < n_chunks && s == LL_OK; ++i) {
      const int slot = (int)(i % nslot);
      char* ds = (char*)dev_src + (size_t)slot * cs;
      char* dd = (char*)dev_dst + (size_t)slot * cs;
      size_t in_off, in_len, out_off, out_len;
      int64_t nb = 1;
      if (n_sh > 1) {
        const int nsh = sched[i].first, idx = sched[i].second;
        in_len = sb / nsh;
        in_off = (size_t)idx * in_len;
        out_len = db / nsh;
        out_off = (size_t)idx * out_len;
      } else {
        const int64_t b0 = i * per_chunk;
        nb = std::min<int64_t>(per_chunk, batch - b0);
        in_off = b0 * sb;
        in_len = nb * sb;
        out_off = b0 * db;
        out_len = nb * db;
      }
      if (i >= nslot) cudaStreamWaitEvent(hp.h2d, hp.ev_comp[slot], 0);
      cudaMemcpyAsync(ds, (const char*)src_host + in_off, in_len, cudaMemcpyHostToDevice, hp.h2d);
      cudaEventRecord(hp.ev_h2d[slot], hp.h2d);
      cudaStreamWaitEvent(hp.comp, hp.ev_h2d[slot], 0);
      if (i >= nslot) cudaStreamWaitEvent(hp.comp, hp.ev_d2h[slot], 0);
      if (n_sh > 1) {
        s = ll_convert_shard(ds, src_layout, dd, dst_layout, elem_bits, sched[i].first, sched[i].second,
                             nullptr, (ll_stream)hp.comp);
      } else {
        ll_convert_options o{};
        o.path = LL_PATH_AUTO;
        o.batch = nb;
        s = ll_convert_ex(ds, src_layout, dd, dst_layout, elem_bits, &o, (ll_stream)hp.comp);
      }
      cudaEventRecord(hp.ev_comp[slot], hp.comp);
      cudaStreamWaitEvent(hp.d2h, hp.ev_comp[slot], 0);
      cudaMemcpyAsync((char*)dst_host + out_off, dd, out_len, cudaMemcpyDeviceToHost, hp.d2h);
      cudaEventRecord(hp.ev_d2h[slot], hp.d2h);
    }
    // the caller's stream resumes after the last copy-out (and the other two
    // streams are drained, so the next call starts from a clean pipeline)
    cudaEventRecord(hp.fin[0], hp.h2d);
    cudaEventRecord(hp.fin[1], hp.comp);
    cudaEventRecord(hp.fin[2], hp.d2h);
    for (int k = 0; k < 3; ++k) cudaStreamWaitEvent(st, hp.fin[k], 0);
    cudaError_t e = cudaStreamSynchronize(st);
    if (s != LL_OK) return s;
    return cuda_status(e, "ll_convert_host");
  });
}

ll_status ll_convert_host_shard(const void* src_host, ll_layout src_layout, void* dst_host,
                                ll_layout dst_layout, int elem_bits, int n_shards, int shard,
                                void* dev_src, void* dev_dst, size_t scratch_bytes, ll_stream stream) {
  return guarded([&]() -> ll_status {
    check_layout(src_layout, "ll_convert_host_shard");
    check_layout(dst_layout, "ll_convert_host_shard");
    const int w = elem_bytes(elem_bits);
    if (!src_host || !dst_host || !dev_src || !dev_dst)
      return fail(LL_ERR_ARG, "ll_convert_host_shard: NULL buffer");
    if (n_shards < 1 || (n_shards & (n_shards - 1)) || shard < 0 || shard >= n_shards)
      return fail(LL_ERR_ARG, "ll_convert_host_shard: n_shards must be a power of two, 0 <= shard < n_shards");
    auto P = ll::get_convert_plan(src_layout->L, dst_layout->L, w, LL_PATH_AUTO, 1);
    ll::shard_range(*P, n_shards, shard);   // throws if not shardable
    const size_t sb = (size_t)w << src_layout->L.in_bits(), db = (size_t)w << dst_layout->L.in_bits();
    const size_t slice = std::max(sb, db) / (size_t)n_shards;
    const int chunk_knob = ll::planner_knob("host_chunk_mb", 0);   // <= 0: the default
    const size_t target = (size_t)(chunk_knob > 0 ? chunk_knob : 32) << 20;
    const size_t cap = std::max<size_t>(1, std::min(target, scratch_bytes));
    // k sub-shards per shard: the smallest power of two whose chunks fit
    int k = 1;
    while (slice / k > cap && k < (1 << 12)) k *= 2;
    while (k > 1) {
      try {
        ll::shard_range(*P, n_shards * k, shard * k);
        break;
      } catch (const ll::Error&) {
        k /= 2;
      }
    }
    const size_t cs = slice / k;
    if (scratch_bytes < cs) return fail(LL_ERR_ARG, "ll_convert_host_shard: scratch smaller than one chunk");
    const int max_slots = std::max(1, std::min(HostPipe::kSlots, ll::planner_knob("host_slots", 2)));
    const int nslot = (int)std::max<size_t>(1, std::min<size_t>(max_slots, scratch_bytes / cs));
    const size_t in_len = sb / ((size_t)n_shards * k), out_len = db / ((size_t)n_shards * k);
    // the sub-shards must tile the shard's slices in order on both sides
    for (int j = 0; j < k; ++j) {
      const ll::TileRange rg = ll::shard_range(*P, n_shards * k, shard * k + j);
      const int64_t q = (int64_t)shard * k + j;
      if (rg.src_shift != q * (int64_t)in_len || rg.dst_shift != q * (int64_t)out_len)
        return fail(LL_ERR_UNSUPPORTED, "ll_convert_host_shard: sub-shards are not contiguous in order");
    }
    // the pipeline of ll_convert_host over this shard's k sub-shards
    HostPipe& hp = host_pipe();
    std::lock_guard<std::mutex> lk(hp.mu);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    cudaEventRecord(hp.start, st);
    cudaStreamWaitEvent(hp.h2d, hp.start, 0);
    cudaStreamWaitEvent(hp.comp, hp.start, 0);
    cudaStreamWaitEvent(hp.d2h, hp.start, 0);
    ll_status s = LL_OK;
    for (int j = 0; j < k && s == LL_OK; ++j) {
      const int slot = j % nslot;
      char* ds = (char*)dev_src + (size_t)slot * cs;
      char* dd = (char*)dev_dst + (size_t)slot * cs;
      if (j >= nslot) cudaStreamWaitEvent(hp.h2d, hp.ev_comp[slot], 0);
      cudaMemcpyAsync(ds, (const char*)src_host + (size_t)j * in_len, in_len, cudaMemcpyHostToDevice, hp.h2d);
      cudaEventRecord(hp.ev_h2d[slot], hp.h2d);
      cudaStreamWaitEvent(hp.comp, hp.ev_h2d[slot], 0);
      if (j >= nslot) cudaStreamWaitEvent(hp.comp, hp.ev_d2h[slot], 0);
      s = ll_convert_shard(ds, src_layout, dd, dst_layout, elem_bits, n_shards * k, shard * k + j, nullptr,
                           (ll_stream)hp.comp);
      cudaEventRecord(hp.ev_comp[slot], hp.comp);
      cudaStreamWaitEvent(hp.d2h, hp.ev_comp[slot], 0);
      cudaMemcpyAsync((char*)dst_host + (size_t)j * out_len, dd, out_len, cudaMemcpyDeviceToHost, hp.d2h);
      cudaEventRecord(hp.ev_d2h[slot], hp.d2h);
    }
    cudaEventRecord(hp.fin[0], hp.h2d);
    cudaEventRecord(hp.fin[1], hp.comp);
    cudaEventRecord(hp.fin[2], hp.d2h);
    for (int q = 0; q < 3; ++q) cudaStreamWaitEvent(st, hp.fin[q], 0);
    cudaError_t e = cudaStreamSynchronize(st);
    if (s != LL_OK) return s;
    return cuda_status(e, "ll_convert_host_shard");
  });
}

ll_status ll_gather_host(const void* src_host, const int32_t* idx_host, void* out_host,
                         ll_layout layout, int axis, int elem_bits, int64_t batch, void* dev_src,
                         void* dev_idx, void* dev_out, size_t scratch_bytes, ll_stream stream) {
  return guarded([&]() -> ll_status {
    check_layout(layout, "ll_gather_host");
    const int w = elem_bytes(elem_bits);
    if (!src_host || !idx_host || !out_host || !dev_src || !dev_idx || !dev_out)
      return fail(LL_ERR_ARG, "ll_gather_host: NULL buffer");
    if (batch < 1) batch = 1;
    const int64_t n = int64_t(1) << layout->L.in_bits();  // elements per instance
    const size_t ub = (size_t)std::max(w, 4) * n;       // the larger of value / index bytes
    if (scratch_bytes < ub) return fail(LL_ERR_ARG, "ll_gather_host: scratch smaller than one instance");
    const int chunk_knob = ll::planner_knob("host_chunk_mb", 0);   // <= 0: the default
    const size_t target = (size_t)(chunk_knob > 0 ? chunk_knob : 16) << 20;
    const int max_slots = std::max(1, std::min(HostPipe::kSlots, ll::planner_knob("host_slots", 2)));
    int64_t per_chunk = (int64_t)std::max<size_t>(1, target / ub);
    per_chunk = std::min<int64_t>(std::min<int64_t>(per_chunk, (int64_t)(scratch_bytes / ub)), batch);
    const int64_t n_chunks = (batch + per_chunk - 1) / per_chunk;
    const size_t cs = (size_t)per_chunk * ub;
    const int nslot = (int)std::max<size_t>(1, std::min<size_t>(max_slots, scratch_bytes / cs));
    // the pipeline of ll_convert_host: values and indices in on the copy-in
    // stream, the gather on the compute stream, results out on the copy-out
    // stream; slot s is reused only after the chunk that last used it is done
    HostPipe& hp = host_pipe();
    std::lock_guard<std::mutex> lk(hp.mu);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    cudaEventRecord(hp.start, st);
    cudaStreamWaitEvent(hp.h2d, hp.start, 0);
    cudaStreamWaitEvent(hp.comp, hp.start, 0);
    cudaStreamWaitEvent(hp.d2h, hp.start, 0);
    ll_status s = LL_OK;
    for (int64_t i = 0; i < n_chunks && s == LL_OK; ++i) {
      const int slot = (int)(i % nslot);
      const int64_t b0 = i * per_chunk, nb = std::min<int64_t>(per_chunk, batch - b0);
      char* ds = (char*)dev_src + (size_t)slot * cs;
      char* di = (char*)dev_idx + (size_t)slot * cs;
      char* dd = (char*)dev_out + (size_t)slot * cs;
      if (i >= nslot) cudaStreamWaitEvent(hp.h2d, hp.ev_comp[slot], 0);
      cudaMemcpyAsync(ds, (const char*)src_host + (size_t)b0 * n * w, (size_t)nb * n * w,
                      cudaMemcpyHostToDevice, hp.h2d);
      cudaMemcpyAsync(di, idx_host + b0 * n, (size_t)nb * n * 4, cudaMemcpyHostToDevice, hp.h2d);
      cudaEventRecord(hp.ev_h2d[slot], hp.h2d);
      cudaStreamWaitEvent(hp.comp, hp.ev_h2d[slot], 0);
      if (i >= nslot) cudaStreamWaitEvent(hp.comp, hp.ev_d2h[slot], 0);
      ll_convert_options o{};
      o.path = LL_PATH_AUTO;
      o.batch = nb;
      s = ll_gather_ex(ds, (const int32_t*)di, dd, layout, axis, elem_bits, &o, (ll_stream)hp.comp);
      cudaEventRecord(hp.ev_comp[slot], hp.comp);
      cudaStreamWaitEvent(hp.d2h, hp.ev_comp[slot], 0);
      cudaMemcpyAsync((char*)out_host + (size_t)b0 * n * w, dd, (size_t)nb * n * w,
                      cudaMemcpyDeviceToHost, hp.d2h);
      cudaEventRecord(hp.ev_d2h[slot], hp.d2h);
    }
    cudaEventRecord(hp.fin[0], hp.h2d);
    cudaEventRecord(hp.fin[1], hp.comp);
    cudaEventRecord(hp.fin[2], hp.d2h);
    for (int k = 0; k < 3; ++k) cudaStreamWaitEvent(st, hp.fin[k], 0);
    cudaError_t e = cudaStreamSynchronize(st);
    if (s != LL_OK) return s;
    return cuda_status(e, "ll_gather_host");
  });
}

}  // extern "C"
