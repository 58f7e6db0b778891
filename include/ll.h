/*
 * ll.h -- C ABI of the B200-native Linear Layouts library (libll_b200.so).
 *
 * Linear Layouts (arXiv 2505.23819): a layout is a linear map over F2 from
 * hardware index bits (reg / lane / warp / block, or a memory "offset") to the
 * bits of logical tensor coordinates (Definition "Linear Layouts", PAPER.md
 * P:316-318).  This library builds layouts from per-dimension bases, composes,
 * inverts and applies them on the host, and converts / gathers device buffers
 * between layouts with hand-written sm_100a kernels.
 *
 * Conventions (readings A1/A2):
 *   - bit vectors are LSB-first (P:305 footnote);
 *   - input dims are listed minor -> major; the flattened input index puts the
 *     first-listed dim at the lowest bits ("reg" lowest);
 *   - output dims are tensor dims dim0..dimN-1 flattened row-major, last dim
 *     fastest;
 *   - a device buffer for layout L holds 2^(sum of L's input bits) elements;
 *     the element at flattened input index h holds tensor element L(h).
 *
 * Errors: every call returns ll_status; LL_OK = 0.  On failure a message is
 * available from ll_last_error() (thread-local, valid until the next call on
 * the same thread).  No call aborts the process.
 *
 * Ownership: layouts are immutable host objects owned by the caller (destroy
 * with ll_layout_destroy).  All device memory is owned by the caller.  The
 * library owns a thread-safe host plan cache and the device constants of each
 * plan; it never allocates device memory on the conversion path.
 *
 * Streams: device work is enqueued on the given stream (a cudaStream_t; NULL
 * = legacy default stream) with no implicit synchronisation.
 */
#ifndef LL_B200_H
#define LL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ll_layout_s* ll_layout;
struct CUstream_st;
typedef struct CUstream_st* ll_stream; /* == cudaStream_t */

typedef enum {
  LL_OK = 0,
  LL_ERR_ARG = 1,             /* bad argument (NULL, size, alignment, range)      */
  LL_ERR_SHAPE = 2,           /* layouts map to different tensors                  */
  LL_ERR_LABEL = 3,           /* dimension names do not match (compose)            */
  LL_ERR_NOT_SURJECTIVE = 4,  /* a layout that must be surjective is not           */
  LL_ERR_NOT_INVERTIBLE = 5,  /* reserved                                           */
  LL_ERR_RANGE = 6,           /* coordinate out of range                            */
  LL_ERR_UNSUPPORTED = 7,     /* valid request the library cannot execute           */
  LL_ERR_CUDA = 8,            /* a CUDA runtime call or launch failed               */
  LL_ERR_OOM = 9              /* host allocation failed                             */
} ll_status;

/* ---------------------------------------------------------------- layouts -- */

/* Create a layout from per-dimension bases (Definition "Linear Layouts",
 * P:316-321; the columns of the matrix as displayed for layout A).
 *   n_in, in_names[n_in], in_bits[n_in]   input dims, minor -> major (e.g.
 *                                          "reg","lane","warp","block", or
 *                                          "offset"); names unique.
 *   n_out, out_names[n_out], out_bits[n_out]  tensor dims dim0..dimN-1.
 *   bases  int64 array of shape [sum(in_bits)][n_out]: row k (k-th input bit,
 *          LSB-first within each input dim, dims in listed order) holds the
 *          output coordinates of that basis vector; an all-zero row is a zero
 *          column (broadcast).  Coordinates must be < 2^out_bits[d].
 *   *out   receives the new layout (caller owns).
 * Limits: sum(in_bits) <= 62, sum(out_bits) <= 62, n_in, n_out <= 16.
 * Errors: LL_ERR_ARG (NULL, duplicate names, bits < 0), LL_ERR_RANGE. */
ll_status ll_layout_create(int n_in, const char* const* in_names, const int* in_bits,
                           int n_out, const char* const* out_names, const int* out_bits,
                           const int64_t* bases, ll_layout* out);

ll_status ll_layout_destroy(ll_layout l);

/* Query sizes: numbers of dims and total bits.  Any pointer may be NULL. */
ll_status ll_layout_info(ll_layout l, int* n_in, int* n_out, int* in_bits_total,
                         int* out_bits_total);

/* Copy out dim names/bits and bases (same formats as ll_layout_create).
 * name buffers: names[i] must have room for 32 chars.  bases: capacity
 * `cap` int64 entries, needs sum(in_bits) * n_out. */
ll_status ll_layout_get(ll_layout l, char (*in_names)[32], int* in_bits, char (*out_names)[32],
                        int* out_bits, int64_t* bases, size_t cap);

/* outer o inner (Definition "Composition"): the matrix is the
 * label-wise product M_outer M_inner.  inner's output dims must equal outer's
 * input dims as a set of (name, bits) (matched by name).  LL_ERR_LABEL
 * otherwise. */
ll_status ll_compose(ll_layout outer, ll_layout inner, ll_layout* out);

/* Right inverse (Definition "Right Inverse"): Gauss-Jordan over
 * F2, pivots in column order, free (slack) variables zero.  The
 * result maps the tensor (input dims = l's output dims listed fastest first,
 * so the flat index is unchanged) to l's input dims (listed major first).
 * LL_ERR_NOT_SURJECTIVE if l is not surjective. */
ll_status ll_invert(ll_layout l, ll_layout* out);

/* Label-wise product (Definition "Product"): block-diagonal;
 * for a shared label a's bits are low, b's high. */
ll_status ll_product(ll_layout a, ll_layout b, ll_layout* out);

/* Left division (Definition "Left Division"): m = [[m1, 0], [0, m2]]
 * label-wise (for every input label, m's first in_size(m1) bits are m1's
 * columns embedded at the low bits of each output dim, and m's other bits
 * have a zero m1 block); *out = m2 = the remaining columns with m1's output
 * bits removed.  Used to decide whether an instruction tile T (vectorised
 * ld/st.shared, ldmatrix/stmatrix) can lower a layout.  Caller
 * owns *out.  LL_ERR_SHAPE when m is not divisible by m1. */
ll_status ll_left_divide(ll_layout m, ll_layout m1, ll_layout* out);

/* Shape-operation transfer functions (Appendix theorem):
 * for an input layout, the output layout for which the shape operation moves
 * no data between hardware indices (every hardware index keeps its value).
 *   ll_transpose   tt.trans: out dim i of the result = out dim perm[i] of l
 *   ll_reshape     tt.reshape: new row-major dims, same element count (flat
 *                  columns unchanged)
 *   ll_expand_dims tt.expand_dims: insert a size-1 dim `name` at `axis`
 *   ll_broadcast   tt.broadcast: size-1 dim `axis` grows to 2^bits; zero
 *                  columns (copies, lowest first) index the new dim, extra
 *                  register bits are added if there are too few copies
 *   ll_join        tt.join: new fastest dim `name` of size 2 held by a new
 *                  register bit 0 (the two values sit in adjacent registers)
 *   ll_split       tt.split: inverse of join (the last dim, size 2, must be
 *                  held by a single register bit)
 * Errors: LL_ERR_ARG (bad permutation / axis / name), LL_ERR_SHAPE (size
 * mismatch), LL_ERR_UNSUPPORTED (split of a dim not held in registers). */
ll_status ll_transpose(ll_layout l, const int* perm, ll_layout* out);
ll_status ll_reshape(ll_layout l, int n_out, const char* const* out_names, const int* out_bits,
                     ll_layout* out);
ll_status ll_expand_dims(ll_layout l, int axis, const char* name, ll_layout* out);
ll_status ll_broadcast(ll_layout l, int axis, int bits, ll_layout* out);
ll_status ll_join(ll_layout l, const char* name, ll_layout* out);
/* Sliced layout: output dim `axis` removed (the layout of a
 * reduction's result along it).  The matrix loses that dim's rows; columns
 * that only reached it become zero (broadcast), and the result is still
 * surjective.  LL_ERR_ARG for a bad axis.  Caller owns *out. */
ll_status ll_slice(ll_layout l, int axis, ll_layout* out);
/* Blocked layout (Appendix proposition): a tensor of rank dims,
 * shape_bits[i] = log2 of dim i; R / T / W = log2 registers / threads /
 * warps per dim with R[i] + T[i] + W[i] = shape_bits[i]; order[0] = the
 * fastest dim.  Input dims reg, lane, warp; output dims dim0..dim{rank-1}.
 * LL_ERR_SHAPE if the sizes do not add up, LL_ERR_ARG for a bad order. */
ll_status ll_blocked(int rank, const int* shape_bits, const int* R, const int* T, const int* W,
                     const int* order, ll_layout* out);
/* mma.sync register / thread tiles (Appendix proposition, reading
 * A8): operand 0 = lhs (A fragment), 1 = rhs (B fragment), 2 = output
 * (accumulator, m16n8); bitwidth 8, 16 or 32.  Input dims reg, lane; output
 * dims dim0 (rows) and dim1 (columns).  Combine with ll_product for warps /
 * repetitions and ll_slice for sliced mma layouts. */
ll_status ll_mma_tile(int operand, int bitwidth, ll_layout* out);
ll_status ll_split(ll_layout l, ll_layout* out);

/* Apply to one point ("w = Av"): in_coords[n_in] -> out_coords[n_out].
 * LL_ERR_RANGE if a coordinate does not fit its dim. */
ll_status ll_apply(ll_layout l, const int64_t* in_coords, int64_t* out_coords);

/* Predicates: distributed, memory, surjective. */
ll_status ll_layout_props(ll_layout l, int* surjective, int* distributed, int* memory);

/* ------------------------------------------------------------ conversion -- */

/* Convert a device buffer from layout src_layout (A) to dst_layout (B): the
 * conversion B^{-1} o A of P:599-611, executed as a pull (A6):
 *     dst[h] = src[X h],  X = A^{-1} o B  (A^{-1} as in ll_invert),
 * for every h < 2^(input bits of B).  For distributed / memory layouts X h is
 * the lowest preimage of B(h) under A.
 *   src, dst   device pointers (caller-owned, must not overlap), 16-byte aligned
 *   elem_bits  8, 16, 32 or 64 (elements are moved as raw bits)
 *   stream     cudaStream_t
 * Errors: LL_ERR_SHAPE (different tensors), LL_ERR_NOT_SURJECTIVE (A),
 * LL_ERR_ARG (NULL / misaligned / elem_bits), LL_ERR_CUDA (launch failed). */
ll_status ll_convert(const void* src, ll_layout src_layout, void* dst, ll_layout dst_layout,
                     int elem_bits, ll_stream stream);

/* Gather along `axis` (tl.gather): one layout L for src, idx and
 * out (each a buffer of 2^(input bits of L) elements):
 *     out[h] = src[h*],  h* = L^{-1}( L(h) with coordinate `axis` := idx[h] ).
 * idx values must lie in [0, 2^out_bits[axis]); they are not checked on the
 * device unless the environment variable LL_GATHER_CHECK=1 is set, in which
 * case out-of-range indices raise LL_ERR_RANGE after a synchronisation. */
ll_status ll_gather(const void* src, const int32_t* idx, void* out, ll_layout layout, int axis,
                    int elem_bits, ll_stream stream);

/* ------------------------------------------------------ extended control -- */

typedef enum {
  LL_PATH_AUTO = 0,      /* planner's choice (cost model): COPY for the
                            identity; SMEM when its plan exchanges >= 8-byte granules
                            (measured fastest once compiled per plan; broadcast layouts: the
                            dedup plan where measured fast); SHUFFLE when the smem plan's
                            granule is <= 4 bytes and the pair is warp-local (elements of
                            <= 4 bytes); else REGPERM when only the low <= 64 bytes of each
                            chunk are permuted; else SMEM; else GENERIC             */
  LL_PATH_COPY = 1,      /* identity quotient: plain copy                          */
  LL_PATH_SMEM = 2,      /* tile through shared memory with the optimal swizzle; by default
                            in a kernel specialised for the plan at run time (NVRTC, every
                            offset and register index a constant; knob smem_jit=0: the
                            generic kernel, which also serves the fused upcast)        */
  LL_PATH_SHUFFLE = 3,   /* warp-local exchange with warp shuffles; by default in a kernel
                            specialised for the plan at run time (NVRTC; knob shuffle_jit=0:
                            the generic kernel)                                      */
  LL_PATH_GENERIC = 4,   /* element-wise pull (any layouts; the slow baseline)     */
  LL_PATH_SMEM_NOSWIZZLE = 5, /* smem path with an unswizzled staging buffer (ablation) */
  LL_PATH_SMEM_ASYNC = 6, /* smem path fed by cp.async (source granules, multi-stage)  */
  LL_PATH_SMEM_PADDED = 7, /* legacy heuristic: unswizzled staging + 16 B pad per 128 B (ablation) */
  LL_PATH_SMEM_TMA = 8,  /* smem path fed by TMA tensor loads (cp.async.bulk.tensor) into a
                            hardware-swizzled image: the 32/64/128-byte swizzle modes are
                            Def. 5 instances; the planner picks the mode and the
                            reader's lanes so the reads are conflict-free.
                            By default a warp-specialised kernel compiled per plan (NVRTC):
                            one producer warp issues the boxes into an mbarrier ring,
                            8 consumer warps read, release the slot (fence.proxy.async +
                            mbarrier arrive) and store; knobs tma_jit (0: the template
                            kernel), tmaj_stages, tmaj_tpc (tiles per group and CTA; < 0:
                            persistent), tmaj_cps, tmaj_k, tmaj_images.
                            LL_ERR_UNSUPPORTED when the source tile needs > 5 box dims. */
  LL_PATH_REGS = 9,      /* register-faithful: threads are the layouts' own lanes / warps (one
                            CTA per block index, each thread's registers contiguous in the
                            buffers), exchange registers -> smem (optimal swizzle) -> registers
                            with stmatrix / ldmatrix where the layout is divisible by their tile
                            (b16 plain and .trans; for 1-byte elements the sm_100a
                            stmatrix.m16n8.trans.b8 / ldmatrix.m16n16.trans.b8 tiles, knob
                            regs_b8), else vectorised st/ld.shared.  Needs reg/lane/warp/block
                            layouts with equal lane (5) and warp (<= 3) bits, identical block
                            columns and elements of <= 4 bytes; else LL_ERR_UNSUPPORTED.
                            Cost model: a warp-local pair whose shuffle exchange needs <= 4
                            rounds (knob regs_shuffle_max_rounds; 0 = never) runs as
                            LL_PATH_REGS_SHUFFLE (measured faster in-kernel on B200). */
  LL_PATH_SMEM_TMA_STORE = 10, /* as SMEM_TMA, and the destination tile is written to a second
                            hardware-swizzled shared-memory image and stored by one TMA tensor
                            store; the readers' lanes (possibly XOR "diagonals" of tile bits)
                            are chosen so reads AND writes are conflict-free.  No thread issues a
                            global load or store. */
  LL_PATH_REGS_SHUFFLE = 11 /* register-faithful warp-shuffle exchange for warp-local
                            pairs ((B^-1 o A)_warp = I), in a kernel specialised for the
                            plan at run time (NVRTC: every register index a compile-time
                            constant); LL_ERR_UNSUPPORTED otherwise. */,
  LL_PATH_REGPERM = 12   /* no exchange between threads (the quotient is the
                            identity outside registers): X = A^{-1} o B permutes only the low
                            q bits of the buffer index (2^q elements <= 64 bytes) and is the
                            identity above, so every thread loads its 2^q-element chunk,
                            permutes it in registers (renames / prmt, compiled per plan) and
                            stores it -- no shared memory, no shuffles.  AUTO takes it
                            unless the smem plan exchanges >= 8-byte granules (measured
                            1-3 % faster there; knob auto_regperm: 2 = always, 0 = never);
                            LL_ERR_UNSUPPORTED when it does not apply. */
} ll_path;

typedef struct {
  int path;          /* ll_path                                                   */
  int64_t batch;     /* >= 1: buffers hold `batch` consecutive copies of the layout */
  int max_ctas;      /* 0 = auto; else cap on the persistent grid                  */
  int reserved[8];
} ll_convert_options;

/* ll_convert with options (NULL = defaults). */
ll_status ll_convert_ex(const void* src, ll_layout src_layout, void* dst, ll_layout dst_layout,
                        int elem_bits, const ll_convert_options* opts, ll_stream stream);

/* Same with gather options (path, batch).  Paths:
 *   LL_PATH_AUTO     measured on B200: the shared-memory gather
 *                    where it applies (the axis unit fits a CTA), else direct
 *   LL_PATH_SHUFFLE  warp-shuffle gather: the axis vectors L^{-1} e_axis lie in
 *                    one warp's registers and lanes (L_warp^axis =
 *                    L_block^axis = 0, in the coalesced mapping: within the low
 *                    log2(16 / elem_bytes) + 9 buffer bits); 2^|L_reg^axis|
 *                    candidate shuffles per output (reading A19); compiled per
 *                    plan (NVRTC)
 *   LL_PATH_SMEM     shared-memory gather: the axis inside an aligned unit
 *                    whose source + indices fit 96 KiB (L_block^axis = 0);
 *                    two cp.async.bulk (source, indices) per unit into a
 *                    2-stage ring, one ld.shared per output; compiled per plan
 *   LL_PATH_GENERIC  direct: source elements read through L1, any layout
 * LL_ERR_UNSUPPORTED when the requested path does not apply.  A compile or
 * module failure of a compiled kernel falls back to the direct kernel. */
ll_status ll_gather_ex(const void* src, const int32_t* idx, void* out, ll_layout layout, int axis,
                       int elem_bits, const ll_convert_options* opts, ll_stream stream);

/* The CUDA source of the compiled gather kernel for (layout, axis, path =
 * LL_PATH_SHUFFLE or LL_PATH_SMEM) into buf (as ll_jit_source); mode bit 1 =
 * the in-kernel timed variant, bit 0 = compile it with NVRTC for sm_100a
 * instead (no device needed) and return {"compiled": true, "cubin_bytes": n}.
 * LL_ERR_UNSUPPORTED if the path does not apply or NVRTC fails. */
ll_status ll_gather_jit_source(ll_layout layout, int axis, int elem_bits, int path, int mode,
                               char* buf, size_t cap, size_t* need);

/* In-kernel timing of the gather exchange (the paper's fig:micro-gather
 * setting: one CTA): one CTA gathers the first unit of the buffers
 * (shuffle: one warp unit = 2^warp_unit_bits elements; smem: one CTA unit),
 * with the exchange -- idx -> source (lane, register) -> shuffles + select, or
 * idx -> ld.shared -- repeated `reps` times on data already in registers /
 * shared memory; thread 0 writes the clock64 cycles of the repeated section
 * to cycles[0] (device pointer).  out receives the gather of that unit.
 * path = LL_PATH_SHUFFLE or LL_PATH_SMEM; errors as ll_gather_ex. */
ll_status ll_gather_timed(const void* src, const int32_t* idx, void* out, ll_layout layout,
                          int axis, int elem_bits, int path, int reps, long long* cycles,
                          ll_stream stream);

/* The scale layout of the mxfp4 upcast:
 * S = P o dst_layout, where dst_layout maps a destination byte's hardware
 * index to its packed-tensor coordinate (m, kb) and P : (m, kb) -> (m, g =
 * kb >> 4) is the projection onto the E8M0 scale tensor [M][K/32] (one scale
 * per 16 packed bytes = 32 fp4 values) -- a linear layout whose columns for
 * kb bits 0-3 are zero (the broadcast of one scale over its 16 bytes).  The
 * upcast reads scales[flatten(S(h))] for destination byte h.  Caller owns
 * *out; LL_ERR_SHAPE unless dst_layout has two output dims and >= 4 kb bits. */
ll_status ll_mxfp4_scale_layout(ll_layout dst_layout, ll_layout* out);

/* Fused mxfp4 dequantisation with the layout conversion (
 * "Software Emulation" / "Data Shuffling"; OCP MX):
 *   packed    u8 buffer in layout src_layout over (m, kb): byte (m, kb) holds
 *             the E2M1 values of k = 2kb (low nibble) and k = 2kb + 1 (high)
 *   scales    E8M0 bytes, row-major [M][K/32] (K = 2 * 2^kb_bits; one scale
 *             per 32 consecutive k, i.e. per 16 packed bytes), 0xFF = NaN
 *   dst_bf16  2 bf16 per byte of dst_layout (the packed image of the bf16
 *             operand layout, e.g. config 5's destination): bf16 element
 *             2h + n holds  e2m1(m, 2kb + n) * 2^(scale[m][kb/16] - 127),
 *             (m, kb) = dst_layout(h); exact (the products are representable
 *             in bf16, subnormals included), overflow -> +-inf, NaN scale ->
 *             NaN.
 * The conversion runs on the smem path (LL_ERR_UNSUPPORTED otherwise); the
 * decode is fused into its store stage (2 GiB written for config 5, as
 * 256-bit sm_100 stores; by default in a kernel compiled for the plan with
 * NVRTC, knob upcast_jit=0: the template kernel).  packed must be 16-byte and
 * dst_bf16 32-byte aligned (LL_ERR_ARG otherwise). */
ll_status ll_mxfp4_upcast(const void* packed, ll_layout src_layout, const uint8_t* scales,
                          void* dst_bf16, ll_layout dst_layout, const ll_convert_options* opts,
                          ll_stream stream);

/* Register-faithful conversion (LL_PATH_REGS) with in-kernel timing: as
 * ll_convert_ex with path LL_PATH_REGS and `batch`, but the register -> smem
 * -> register exchange is repeated `reps` (>= 1) times inside the kernel and
 * thread 0 of CTA c writes the clock64 cycles of the repeated section to
 * cycles[c] (device buffer of >= min(n_tiles, grid) entries, or NULL), the
 * paper's in-kernel view of a conversion (microbenchmarks: one CTA).
 * dst receives the conversion (identical for every reps).  Errors as
 * ll_convert_ex; LL_ERR_UNSUPPORTED if the layouts are not regs-compatible. */
ll_status ll_convert_regs_timed(const void* src, ll_layout src_layout, void* dst,
                                ll_layout dst_layout, int elem_bits, int64_t batch, int reps,
                                long long* cycles, ll_stream stream);

/* The CUDA source of a run-time specialised kernel for (src_layout,
 * dst_layout) into buf (cap bytes, NUL-terminated; *need = the size needed):
 * the LL_PATH_REGS_SHUFFLE kernel, or with (compile & 2) the LL_PATH_SHUFFLE
 * HBM kernel, (compile & 4) the LL_PATH_SMEM kernel, (& 8) the fused mxfp4
 * upcast, (& 16) the LL_PATH_REGPERM kernel, (& 32 / & 64) the warp-
 * specialised TMA kernels of LL_PATH_SMEM_TMA / LL_PATH_SMEM_TMA_STORE.  (compile & 1) instead compiles it with NVRTC for sm_100a (no
 * device needed) and returns {"compiled": true, "cubin_bytes": n}.
 * LL_ERR_UNSUPPORTED if the pair has no such plan or NVRTC fails. */
ll_status ll_jit_source(ll_layout src_layout, ll_layout dst_layout, int elem_bits, int compile,
                        char* buf, size_t cap, size_t* need);

/* The same for path LL_PATH_REGS (shared memory, repeats A -> B) or
 * LL_PATH_REGS_SHUFFLE (warp shuffles; each repetition converts A -> B -> A
 * so the data are loop-carried, i.e. `reps` repetitions are 2 * reps
 * conversions).  LL_ERR_ARG for any other path. */
ll_status ll_convert_inkernel_timed(const void* src, ll_layout src_layout, void* dst,
                                    ll_layout dst_layout, int elem_bits, int64_t batch, int path,
                                    int reps, long long* cycles, ll_stream stream);

/* Multi-GPU shard: convert only shard `shard` of `n_shards`
 * (a power of two).  The tensor is split along the top log2(n_shards) index
 * bits, which must be block bits shared by both layouts (X maps them
 * identically), so shard s is the contiguous byte range
 *   src: [s * S_A, (s+1) * S_A),  dst: [s * S_B, (s+1) * S_B),
 *   S_A = (elem_bytes << in_bits(A)) / n_shards, S_B likewise,
 * and src_slice / dst_slice point at those ranges in the caller's (e.g. this
 * rank's) memory.  No collective: ranks run independently.
 * Errors: LL_ERR_UNSUPPORTED if the layouts cannot be sharded that way,
 * LL_ERR_ARG for a bad shard index; otherwise as ll_convert_ex. */
ll_status ll_convert_shard(const void* src_slice, ll_layout src_layout, void* dst_slice,
                           ll_layout dst_layout, int elem_bits, int n_shards, int shard,
                           const ll_convert_options* opts, ll_stream stream);

/* Byte ranges of shard `shard`: out4 = {src_begin, src_end, dst_begin, dst_end}. */
ll_status ll_shard_describe(ll_layout src_layout, ll_layout dst_layout, int elem_bits, int path,
                            int n_shards, int shard, int64_t* out4);

/* End-to-end gather of HOST buffers (as ll_gather_ex with
 * `batch` instances of `layout`): src_host (elem_bits values), idx_host
 * (int32, one per output element) and out_host are host pointers (pinned for
 * full speed), chunked by whole instances (~16 MiB, knob "host_chunk_mb")
 * and pipelined like ll_convert_host over the caller's device scratch
 * dev_src / dev_idx / dev_out of scratch_bytes each (>= one instance's
 * max(elem_bytes, 4) * 2^in_bits bytes).  Synchronous. */
ll_status ll_gather_host(const void* src_host, const int32_t* idx_host, void* out_host,
                         ll_layout layout, int axis, int elem_bits, int64_t batch, void* dev_src,
                         void* dev_idx, void* dev_out, size_t scratch_bytes, ll_stream stream);

/* Pitched shard (used by ll_convert_host for layouts that have no
 * contiguous-on-both-sides split, e.g. a transpose): shard `shard` of
 * `n_shards` (a power of two >= 2) is a contiguous slice of one buffer and,
 * in the other, the elements whose index bits [r0, r0 + log2 n_shards) equal
 * `shard` -- rows of elem_bytes << r0 bytes at a pitch of n_shards times
 * that.  out6 = {side (0: src contiguous / dst pitched, 1: the reverse), r0,
 * contiguous-side begin, end (bytes), pitched-side row bytes, pitch bytes}.
 * LL_ERR_UNSUPPORTED when the plan's top tile bits do not allow it. */
ll_status ll_shard_describe_2d(ll_layout src_layout, ll_layout dst_layout, int elem_bits, int path,
                               int n_shards, int shard, int64_t* out6);

/* Checksum of a device buffer (untimed; ours -- the
 * paper has no such step): the 64-bit sum, mod 2^64, over elements h of
 *     fmix( v_h + (index_base + h + 1) * 0x9E3779B97F4A7C15 )     (indexed)
 *     fmix( v_h )                                                  (!indexed)
 * where v_h is element h zero-extended to 64 bits and fmix is the splitmix64
 * output function (z ^= z >> 30; z *= 0xBF58476D1CE4E5B9; z ^= z >> 27;
 * z *= 0x94D049BB133111EB; z ^= z >> 31).  Indexed sums see misplaced
 * elements; the sums of a partition's pieces (index_base = the piece's first
 * element) add up to the whole buffer's.  The index-free sum is invariant
 * under any permutation (a full-size property of bijective conversions).
 *   buf        n_elems elements of elem_bits (8/16/32/64), 16-byte aligned
 *   result     DEVICE pointer to one uint64; overwritten (zeroed, then
 *              accumulated) on `stream`; read it after the stream completes
 * Errors: LL_ERR_ARG (NULL / misaligned / elem_bits / n_elems < 0). */
ll_status ll_checksum(const void* buf, int64_t n_elems, int elem_bits, int indexed,
                      int64_t index_base, uint64_t* result, ll_stream stream);

/* End-to-end conversion of HOST buffers: src_host/dst_host are host pointers
 * (pinned for full speed); the library pipelines host->device copies, the
 * conversion and device->host copies in chunks (16-32 MiB: whole layout
 * instances, or shards of a single large instance -- contiguous in both
 * buffers, else contiguous in one and pitched in the other (ll_shard_describe_2d;
 * the pitched side is then staged whole in its scratch buffer and copied
 * with 2-D copies of >= 1 KiB rows)) over a copy-in, a compute
 * and a copy-out stream of its own, rotating 2 slots (knob: up to 4) of the caller's
 * device scratch buffers dev_src/dev_dst of scratch_bytes each (>= one
 * chunk).  Ordered after work already queued on `stream`; synchronous:
 * returns when dst_host is complete.  Knobs (ll_tune): "host_chunk_mb",
 * "host_slots", "host_2d" (1: pitched shards allowed), "host_ramp" (0; R > 0:
 * the first and last shard chunks cut into 1/2^R .. 1/2 pieces). */
ll_status ll_convert_host(const void* src_host, ll_layout src_layout, void* dst_host,
                          ll_layout dst_layout, int elem_bits, int64_t batch, void* dev_src,
                          void* dev_dst, size_t scratch_bytes, ll_stream stream);

/* End-to-end conversion of ONE RANK'S SHARD from host buffers (SURVEY 8(e):
 * the multi-GPU path with its host copies): src_host holds this shard's
 * source slice and dst_host receives its destination slice -- the byte
 * ranges ll_shard_describe(n_shards, shard) reports, as contiguous host
 * buffers (pinned for full speed).  The slice is cut into k sub-shards
 * (shards n_shards*k, shard*k .. shard*k+k-1; chunks of ~host_chunk_mb)
 * pipelined like ll_convert_host through the caller's device scratch
 * dev_src / dev_dst of scratch_bytes each (>= one chunk).  LL_ERR_UNSUPPORTED
 * when the plan is not shardable; synchronous. */
ll_status ll_convert_host_shard(const void* src_host, ll_layout src_layout, void* dst_host,
                                ll_layout dst_layout, int elem_bits, int n_shards, int shard,
                                void* dev_src, void* dev_dst, size_t scratch_bytes, ll_stream stream);

/* JSON description of the plan the planner builds for (src, dst, elem_bits)
 * with the given path request: path, tile bits, thread mapping, granule,
 * swizzle bases, predicted wavefronts, shuffle sets.  Writes at most cap bytes
 * (NUL-terminated); *needed receives the full length. */
ll_status ll_plan_describe(ll_layout src_layout, ll_layout dst_layout, int elem_bits, int path,
                           char* json, size_t cap, size_t* needed);

/* Gather-plan description (same conventions). */
ll_status ll_gather_describe(ll_layout layout, int axis, int elem_bits, int path, char* json,
                             size_t cap, size_t* needed);

/* Number of kernel launches issued by this library since load (for the
 * benchmark's gpu_launches claim). */
int64_t ll_launch_count(void);

/* Tuning knobs (process-wide).  Launch configuration (defaults from the
 * environment, read once):
 *   "tpg"        target tiles per tile group of the smem kernel (0 = persistent
 *                grid at full occupancy; env LL_TPG, default 2)
 *   "pipe"       1 = software-pipelined smem kernel (env LL_PIPE, default 1)
 *   "up_tpg"     tiles per group of the mxfp4 upcast kernel (env LL_UP_TPG,
 *                default 0 = persistent)
 *   "gather_vpt" 16-byte output vectors per thread of the gather kernels
 *                (env LL_GATHER_VPT; 0 = per path: shuffle 4, direct 1)
 *   "gather_shfl_u" warp-vectors whose loads the shuffle gather issues
 *                before its first shuffle (1, 2 or 4; default 2)
 *   "carveout", "pow2", "stages", "async_tpg"  ablation knobs of the smem /
 *                cp.async kernels (env LL_CARVEOUT, LL_POW2, LL_STAGES,
 *                LL_ASYNC_TPG)
 * Planner (new plans only; cached plans are rebuilt):
 *   "thread_bytes", "thread_bytes_max", "max_granule", "run_bytes",
 *   "tile_order"  thread vector bytes, granule cap, coalescing run bytes,
 *                tile index order
 * Executors compiled per plan (NVRTC; jit.cpp):
 *   "smem_jit" (1) / "shuffle_jit" (1) / "upcast_jit" (1)  compile the plan
 *                (0 = the template kernels); "smem_jit_tpg" (1),
 *                "shuffle_jit_tpg" (1), "upcast_jit_tpg" (4) tiles per group;
 *                "smem_jit_minb" (0 = auto) register cap; "smem_jit_depth"
 *                (1) tiles in flight; "smem_jit_single" (0) one staging
 *                buffer per group when each group has one tile; "pdl" (1)
 *                programmatic dependent launch;
 *                "jit_force_fail" (0) test hook
 *   "auto_shuffle" (0)  AUTO prefers the compiled shuffle exchange when the
 *                warp tile is warp-local
 * TMA paths: "tma_tpg" (-1 = by wave count), "tma_stages" (3),
 *   "tma_run_bytes" (256), "tma_thread_bytes" (64), "tma_tile_bytes" (8192),
 *   "tma_force_swizzle" (-1)
 * Session-3 knobs: "pdl_prefetch" (1: the first wave of the
 *   compiled smem kernel prefetches its first tile's source into L2 before
 *   griddepcontrol.wait; 2: every CTA; 0: off), "pdl_prefetch_waves" (2:
 *   also the tiles of the CTAs replacing it in wave 2; "shuffle_prefetch_waves" (3)
 *   the same for the shuffle kernel), "pdl_prefetch_short" (0),
 *   "gather_prefetch_waves" (1: the smem gather's first wave bulk-prefetches its
 *   units), "shuffle_pdl" (1) / "gather_pdl" (1) / "upcast_pdl" (0) programmatic
 *   dependent launch of those kernels, "regperm_prefetch" (0),
 *   "auto_regperm_shuffle" (1: AUTO takes the warp-shuffle exchange over the
 *   register permutation where it applies), "ld_hint" / "st_hint" (0: global
 *   cache-qualifier ablation), "tile_xor" (0) / "tile_xor_skip" (1) diagonal
 *   tile order, "gather_auto_smem" (1: AUTO smem gather wherever it fits)
 * Register-faithful paths: "regs_matrix" (1) stmatrix / ldmatrix allowed,
 *   "regs_trans" (1) their .trans forms, "regs_shuffle_max_rounds" (4)
 * ll_convert_host: "host_chunk_mb" (default: 32 for shards of one instance, 16
 *   for whole instances and pitched shards; ll_gather_host 16), "host_slots"
 *   (default 2), "host_ramp" (default 0).
 * LL_ERR_ARG for an unknown name.  Used by the tuning sweeps. */
ll_status ll_tune(const char* name, int value);

const char* ll_last_error(void);

/* Library version string. */
const char* ll_version(void);

#ifdef __cplusplus
}
#endif
#endif /* LL_B200_H */
