// kernels.hpp -- host launchers of the sm_100a kernels (kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include "plan.hpp"

namespace ll {

// w = element bytes, nv = 16-byte vectors per thread per side, g = granule bytes.
cudaError_t launch_convert_smem(const SmemPlan& p, int w, int nv, int g, const void* src,
                                void* dst, int max_ctas, cudaStream_t st, const TileRange& rg);
cudaError_t launch_convert_shuffle(const ShufflePlan& p, int w, int nv, const void* src, void* dst,
                                   int max_ctas, cudaStream_t st, const TileRange& rg);
cudaError_t launch_convert_async(const SmemPlan& p, int w, int nv, const void* src, void* dst,
                                 int max_ctas, cudaStream_t st, const TileRange& rg);
cudaError_t launch_convert_tma(const SmemPlan& p, const TmaDesc& td, int w, int nv,
                               const void* src, void* dst, int max_ctas, cudaStream_t st,
                               const TileRange& rg);
cudaError_t launch_convert_tma_store(const SmemPlan& p, const TmaDesc& tds, const TmaDesc& tdd,
                                     int w, int nv, const void* src, void* dst, int max_ctas,
                                     cudaStream_t st, const TileRange& rg);
// Tensor map (128-byte CUtensorMap at tm) of a TmaDesc view of base[0, slice_elems).
cudaError_t encode_tma_map(void* tm, const TmaDesc& td, int w, const void* base, int64_t slice_elems);
cudaError_t launch_convert_regs(const RegsPlan& p, int w, const void* src, void* dst,
                                int max_ctas, int reps, long long* cycles, cudaStream_t st);
cudaError_t launch_convert_generic(const GenericPlan& p, int w, const void* src, void* dst,
                                   int max_ctas, cudaStream_t st);
cudaError_t launch_gather(const GatherPlan& p, int w, bool shuffle, const void* src,
                          const int32_t* idx, void* out, int* err, int max_ctas, cudaStream_t st);
cudaError_t launch_mxfp4_upcast(const SmemPlan& p, int nv, int g, const void* src, void* dst,
                                const uint8_t* scales, int max_ctas, cudaStream_t st,
                                const TileRange& rg);
cudaError_t launch_checksum(const void* buf, int64_t n, int w, bool indexed, int64_t base,
                            unsigned long long* result, cudaStream_t st);
int device_sm_count();
int set_knob(const char* name, int value);

}  // namespace ll
