// K4 — chunked-prefill paged attention on the 5th-generation tensor cores
// (tcgen05 / TMEM), SURVEY §8f-3. The reference computes no attention at all
// (SPEC.md:278); its engine::step allocates one prefill chunk per iteration
// (engine.cpp:182-210) and this kernel is the attention of that chunk:
//
//   for each query token i of the chunk (absolute position p_i = first + i)
//   and q head h:  O[i][h] = softmax(q·Kᵀ · scale) · V over the request's
//   keys 0..p_i (causal), K/V read from the pool's pages through the block
//   table, kv head h / G (GQA).
//
// Work decomposition. The G q heads of a kv head are packed into the MMA's M
// dimension: Q-tile row r = token (r / G) x head (r % G), 128 rows =
// floor(128 / G) tokens. A UNIT is a pair of consecutive Q tiles of one kv
// head (256 rows) over the key tiles (64 keys) the pair may attend; each
// K/V tile a CTA loads feeds BOTH Q tiles (half the K/V gather per FLOP of a
// one-tile CTA). The units' key tiles are concatenated (kv head major) and
// cut stream-K style into equal contiguous ranges, one per CTA (grid = SM
// count, one CTA per SM): no wave tail, and causal units of unequal length
// balance. A unit cut by range boundaries leaves one fp32 partial (O, m, l)
// per CTA; the LAST CTA to publish its partial (ticket per unit) merges them
// — no CTA ever waits for another, so any residency makes progress.
//
// Warp roles (512 threads, one CTA per SM; TMEM: S0 buffers 0/1 | S1 buffers
// 0/1 (64 columns each) | O0 | O1; setmaxnreg moves registers from the loader
// / MMA warpgroups to the softmax ones):
//   warps 0-3   softmax warpgroup 0 (Q tile 0 of the unit): thread r owns
//               row r = TMEM lane r; reads an S0 buffer with one tcgen05.ld,
//               online softmax in the log2 domain with lazy rescaling (O0
//               rescaled in TMEM only when a row max grows by more than 2^8),
//               writes P0 (bf16) back into the buffer's columns, epilogue
//               O0 / l (or a partial);
//   warps 4-7   softmax warpgroup 1: the same for Q tile 1 (S1, O1);
//   warps 10-11 loaders (warps 8-9 idle, so the two schedulers of the MMA
//               warps carry no loader): Q pair once per unit segment, then each 64-key K
//               and V tile gathered from the pages with cp.async (16 B per
//               thread-op) into 128B-swizzled tiles (the UMMA canonical
//               layout) through a ring of K|V halves; every thread owns a
//               fixed tile row and decodes its slot id one tile ahead, and
//               publishes its copies itself (cp.async group wait, proxy
//               fence, mbarrier arrive, a few groups behind the issue);
//   warps 12-13 TMEM allocation (12); warp 12 + j issues every tcgen05.mma of
//               Q tile j: S_j(t) into one of two S buffers, two tiles ahead
//               of O_j += P_j(t)·V(t), so the softmax of tile t+1 never
//               waits for the MMAs of tile t. P(t) aliases its S buffer in
//               TMEM: the MMAs of one thread execute in issue order, so
//               S(t+2) overwrites P(t) only after P(t)·V(t) read it. Warps
//               14-15 only give their registers away.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "cuda/attn_common.cuh"
#include "cuda/device_impl.cuh"

namespace prism {

namespace {

struct PrefillArgs {
    KvGeom g;
    int layer;
    const __nv_bfloat16* q;   // [chunk][n_q][D]
    __nv_bfloat16* out;       // [chunk][n_q][D]
    const std::int32_t* row;  // block-table row of the request (slot ids in token order)
    int first;                // absolute position of the chunk's first token
    int chunk;                // query tokens
    float scale_log2;
    float rescale_thr;        // lazy-rescale threshold (log2 units; 8)
    int merge_fast;           // 1: merges of <= 4 parts issue all their loads at once (PRISM_K4_MERGE)
    int perm;                 // 1: CTA b takes range b / 2 (even b) or ceil(grid / 2) + b / 2 (odd b) (PRISM_K4_PERM)
    int early_ticket;         // 1: a mid-range partial's ticket is a release atomic checked at the next epilogue (PRISM_K4_EARLY)
    int tab_smem;             // 1: the pair prefix is read from a shared-memory copy when it fits (PRISM_K4_TAB=0: global)
    int n_qp;                 // Q-tile pairs per kv head
    const std::int32_t* qp_tiles;  // [n_qp + 1] key-tile prefix over the pairs (same for every kv head)
    int per_cta;              // key tiles per CTA range
    int total;                // key tiles of all units = n_kv * qp_tiles[n_qp]
    uint2* part_o;            // [2 * grid][D / 4][256] O / l of cut units, fp16 x 4
    float2* part_ml;          // [2 * grid][256] (m, l) of cut units
    int* tickets;             // [n_kv * n_qp], zero between launches
    unsigned long long* trace;  // PRISM_K4_TRACE: [13][1024] globaltimer stamps of one CTA, else null
    int trace_cta;            // the traced CTA (PRISM_K4_TRACE_CTA, default 0)
    unsigned long long* cta_trace;  // PRISM_K4_CTA_TRACE: [grid][4] stamps of this launch, else null
    unsigned* dbg;            // PRISM_K4_DEBUG: host-mapped progress words (CTA 0 only), else null
};

// timeline stamp (no-op unless PRISM_K4_TRACE): role 0 loader issued tile t,
// 1 S(t) issued (both Q tiles), 2 / 7 P0(t)·V(t) / P1(t)·V(t) issued,
// 3 / 5 warpgroup 0 / 1 has S(t), 4 / 6 it posted P(t)
__device__ __forceinline__ void k4_stamp(unsigned long long* tr, int cta, int role, int t) {
    if (tr && static_cast<int>(blockIdx.x) == cta && t < 1024) {
        unsigned long long ns;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
        tr[role * 1024 + t] = ns;
    }
}

// per-CTA launch timeline (no-op unless PRISM_K4_CTA_TRACE): 0 CTA start,
// 1 the SM id, 2 first-write PDL wait returned (softmax thread 0), 3 CTA end
__device__ __forceinline__ void k4_cta_stamp(unsigned long long* tr, int k) {
    if (tr) {
        unsigned long long ns;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
        tr[blockIdx.x * 4 + k] = ns;
    }
}

// progress marker for hang diagnosis (no-op unless PRISM_K4_DEBUG)
__device__ __forceinline__ void k4_mark(unsigned* dbg, int slot, unsigned v) {
    if (dbg && blockIdx.x == 0) {
        *reinterpret_cast<volatile unsigned*>(dbg + slot) = v;
        __threadfence_system();
    }
}

template <int D>
struct PfShape {
    static constexpr int kM = 128;            // MMA rows per Q tile (packed token x head)
    static constexpr int kN = 64;             // keys per K/V tile
    static constexpr int kQB = kM * D * 2;    // one Q tile
    static constexpr int kHalfB = kN * D * 2;  // one K (or V) tile
    static constexpr int kHalves = D == 128 ? 6 : 16;  // ring slots of K|V halves
    static constexpr int kOffQ = 0;           // Q pair buffers 0 and 1 (tiles 0, 1 each)
    static constexpr int kOffKV = 4 * kQB;
    static constexpr int kOffBar = kOffKV + kHalves * kHalfB;
    // q_full[2] | q_empty[2] | kv_full[H] | kv_empty[H] | s_full[2][2] | p_full[2][2] | pv_done[2][2] | o_free[2]
    static constexpr int kBars = 4 + 2 * kHalves + 14;
    static constexpr int kOffMisc = kOffBar + kBars * 8;  // TMEM address, merge flag
    static constexpr int kOffTab = kOffMisc + 16;         // qp_tiles prefix (when n_qp < kMaxTab)
    static constexpr int kMaxTab = 384;
    static constexpr int kSmem = kOffTab + kMaxTab * 4 + 1024;  // + alignment slack
    static constexpr int kThreads = 512;
    static constexpr int kLoaders = 64;       // warps 10-11 (schedulers 2, 3; the MMA warps own 0, 1)
    // setmaxnreg split of the 64K registers: softmax warpgroups 0-1 grow,
    // loader warpgroup 2 and the MMA warpgroup 3 shrink (2 x 128 x (168 + 88))
    static constexpr int kRegsSoftmax = 168;
    static constexpr int kRegsLoad = 88;
    static constexpr std::uint32_t kTmemCols = 512;
    static constexpr std::uint32_t kColO = 256;  // S0 buffers 0/1, S1 buffers 0/1 (kN each), O0, O1
};
static_assert(PfShape<128>::kSmem <= 232448, "K4 shared memory");

// ---------------------------------------------------------------- PTX helpers
// High word of every shared-memory matrix descriptor used here: SBO 1024 B
// (8-row groups), descriptor version 1 (sm_100), SWIZZLE_128B.
constexpr std::uint32_t kDescHi = (1024u >> 4) | (1u << 14) | (2u << 29);
__device__ __forceinline__ std::uint32_t saddr(const void* p) {
    return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mb_init(std::uint32_t bar, std::uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ bool mb_try(std::uint32_t bar, std::uint32_t parity) {
    std::uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mb_wait(std::uint32_t bar, std::uint32_t parity) {
    while (!mb_try(bar, parity)) {
    }
}
__device__ __forceinline__ void mb_arrive(std::uint32_t bar) {
    std::uint64_t st;
    asm volatile("mbarrier.arrive.shared::cta.b64 %0, [%1];\n" : "=l"(st) : "r"(bar) : "memory");
    (void)st;
}
// arrives on `bar` once all of this thread's earlier cp.async copies landed
// (does not block the thread; the arrival counts against the init count)
__device__ __forceinline__ void cp_async_arrive(std::uint32_t bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(bar) : "memory");
}
// 16-byte cp.async to a shared-window address (src_bytes 0: zero fill)
__device__ __forceinline__ void cp_async16_s(std::uint32_t dst, const void* src, int src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(src_bytes));
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
// tcgen05 ops issued warp-wide: every lane executes them with the same
// operands and one elected lane issues (no divergent single-lane region
// around the uniform ops). MMAs are kind::f16: bf16 in, fp32 accumulate.
__device__ __forceinline__ void tc_commit_e(std::uint32_t bar) {
    asm volatile(
        "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
        " @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(bar)
        : "memory");
}
// One tile's MMAs from one asm statement (the operands reach the uniform
// datapath once; per-MMA descriptors are 64-bit adds of the low word inside):
// S_j = Q_j · K(k)ᵀ over head_dim in K=16 steps (+32 B inside a 128-byte
// atom, next atom 128 Q rows / 64 K rows further), fresh accumulator.
template <int D>
__device__ __forceinline__ void tc_mma_s_tile(std::uint32_t d_tmem, std::uint64_t dq, std::uint64_t dk,
                                              std::uint32_t idesc) {
    static_assert(D == 64 || D == 128, "head_dim");
    if constexpr (D == 128) {
        asm volatile(
        "{\n .reg .pred e, f, t;\n .reg .b64 a, b;\n setp.ne.b32 t, 1, 0;\n setp.ne.b32 f, 1, 1;\n elect.sync _|e, 0xffffffff;\n"
        " add.s64 a, %1, 0;\n add.s64 b, %2, 0;\n"
        " @e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, f;\n"
        " add.s64 a, %1, 2;\n add.s64 b, %2, 2;\n"
        " @e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n"
        " add.s64 a, %1, 4;\n add.s64 b, %2, 4;\n"
        " @e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n"
        " add.s64 a, %1, 6;\n add.s64 b, %2, 6;\n"
        " @e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n"
        " add.s64 a, %1, 1024;\n add.s64 b, %2, 512;\n"
        " @e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n"
        " add.s64 a, %1, 1026;\n add.s64 b, %2, 514;\n"
        " @e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n"
        " add.s64 a, %1, 1028;\n add.s64 b, %2, 516;\n"
        " @e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n"
        " add.s64 a, %1, 1030;\n add.s64 b, %2, 518;\n"
        " @e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n"
        "}\n"
        ::"r"(d_tmem), "l"(dq), "l"(dk), "r"(idesc)
        : "memory");
    } else {
        asm volatile(
        "{\n .reg .pred e, f, t;\n .reg .b64 a, b;\n setp.ne.b32 t, 1, 0;\n setp.ne.b32 f, 1, 1;\n elect.sync _|e, 0xffffffff;\n"
        " add.s64 a, %1, 0;\n add.s64 b, %2, 0;\n"
        " @e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, f;\n"
        " add.s64 a, %1, 2;\n add.s64 b, %2, 2;\n"
        " @e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n"
        " add.s64 a, %1, 4;\n add.s64 b, %2, 4;\n"
        " @e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n"
        " add.s64 a, %1, 6;\n add.s64 b, %2, 6;\n"
        " @e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n"
        "}\n"
        ::"r"(d_tmem), "l"(dq), "l"(dk), "r"(idesc)
        : "memory");
    }
}
// O_j (+)= P_j · V(k) over the tile's 64 keys in K=16 steps: P (the A
// operand) from tensor memory, lane = row, two bf16 K-elements per 32-bit
// column (+8 columns per step); V MN-major (+16 rows = 2048 B per step).
__device__ __forceinline__ void tc_mma_pv_tile(std::uint32_t d_tmem, std::uint32_t p_tmem, std::uint64_t dv,
                                               std::uint32_t idesc, std::uint32_t accumulate) {
    asm volatile(
        "{\n .reg .pred e, p, t;\n .reg .b64 b;\n .reg .b32 a;\n setp.ne.b32 t, 1, 0;\n setp.ne.b32 p, %4, 0;\n elect.sync _|e, 0xffffffff;\n"
        " add.s32 a, %1, 0;\n add.s64 b, %2, 0;\n"
        " @e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, p;\n"
        " add.s32 a, %1, 8;\n add.s64 b, %2, 128;\n"
        " @e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, t;\n"
        " add.s32 a, %1, 16;\n add.s64 b, %2, 256;\n"
        " @e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, t;\n"
        " add.s32 a, %1, 24;\n add.s64 b, %2, 384;\n"
        " @e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, t;\n"
        "}\n"
        ::"r"(d_tmem), "r"(p_tmem), "l"(dv), "r"(idesc), "r"(accumulate)
        : "memory");
}
// 32 consecutive fp32 columns of this thread's TMEM lane
__device__ __forceinline__ void tc_ld32(std::uint32_t taddr, float (&v)[32]) {
    std::uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tc_st32(std::uint32_t taddr, const float (&v)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
        "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};\n" ::"r"(
            taddr),
        "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
        "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
        "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
        "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
        "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
        "r"(__float_as_uint(v[15])), "r"(__float_as_uint(v[16])), "r"(__float_as_uint(v[17])),
        "r"(__float_as_uint(v[18])), "r"(__float_as_uint(v[19])), "r"(__float_as_uint(v[20])),
        "r"(__float_as_uint(v[21])), "r"(__float_as_uint(v[22])), "r"(__float_as_uint(v[23])),
        "r"(__float_as_uint(v[24])), "r"(__float_as_uint(v[25])), "r"(__float_as_uint(v[26])),
        "r"(__float_as_uint(v[27])), "r"(__float_as_uint(v[28])), "r"(__float_as_uint(v[29])),
        "r"(__float_as_uint(v[30])), "r"(__float_as_uint(v[31]))
        : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
}

// 64 consecutive fp32 columns of this thread's TMEM lane, one load + wait
// (the outputs are defined by the same asm statement as the wait)
__device__ __forceinline__ void tc_ld64(std::uint32_t taddr, float (&v)[64]) {
    std::uint32_t r[64];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32, %33, %34, %35, %36, %37, %38, %39, %40, %41, %42, %43, %44, %45, %46, %47, %48, %49, %50, %51, %52, %53, %54, %55, %56, %57, %58, %59, %60, %61, %62, %63}, [%64];\n"
        "tcgen05.wait::ld.sync.aligned;\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]), "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]), "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]), "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
        : "r"(taddr)
        : "memory");
#pragma unroll
    for (int i = 0; i < 64; ++i) v[i] = __uint_as_float(r[i]);
}
// 32 consecutive 32-bit columns of this thread's TMEM lane (no wait)
__device__ __forceinline__ void tc_st32_nowait(std::uint32_t taddr, const std::uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
        "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};\n" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
        "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
        "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
        "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
        : "memory");
}

__device__ __forceinline__ std::uint32_t pack_f16(float lo, float hi) {
    const __half2 p = __floats2half2_rn(lo, hi);
    return *reinterpret_cast<const std::uint32_t*>(&p);
}
__device__ __forceinline__ float2 unpack_f16(std::uint32_t w) {
    return __half22float2(*reinterpret_cast<const __half2*>(&w));
}

// Shared-memory matrix descriptor (sm_100 "version 1"), 128-byte swizzle.
// K-major canonical layout ((8,m),(T,2)):((8T,SBO),(1,T)): rows of 128 B,
// 8-row groups 1024 B apart (SBO), LBO unused (1). MN-major canonical layout
// ((T,8,n),(8,k)):((1,T,LBO),(8T,SBO)): 64-element atoms along MN `lbo` bytes
// apart, 8-row K groups 1024 B apart.
// Fields: start address >> 4 (bits 0-13), LBO >> 4 (16-29), SBO >> 4 = 64
// (32-45), version 1 (46), SWIZZLE_128B (61-63).
// Its low word (start address >> 4, LBO >> 4) varies
// per operand tile and K step and never carries into the high word (shared
// addresses < 256 KB), which is the constant kDescHi. Offsets are added to the
// low word as >> 4.
__device__ __forceinline__ std::uint32_t desc_lo(std::uint32_t addr, std::uint32_t lbo_bytes) {
    return ((addr >> 4) & 0x3fffu) | (((lbo_bytes >> 4) & 0x3fffu) << 16);
}
__device__ __forceinline__ std::uint64_t desc_of(std::uint32_t lo) {
    return (static_cast<std::uint64_t>(kDescHi) << 32) | lo;
}
// Instruction descriptor, kind::f16: bf16 A/B, fp32 D, M x N, K-major A,
// B K-major (b_mn = 0) or MN-major (b_mn = 1).
__host__ __device__ constexpr std::uint32_t f16_idesc(int m, int n, int b_mn) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<std::uint32_t>(b_mn) << 16) |
           (static_cast<std::uint32_t>(n >> 3) << 17) | (static_cast<std::uint32_t>(m >> 4) << 24);
}
// Byte offset of 16-byte chunk `c` (of a row of D/8 chunks) of tile row `r`
// in a K-major 128B-swizzled tile made of D/64 atoms of rows x 128 B.
template <int ROWS>
__device__ __forceinline__ std::uint32_t sw_off(int r, int c) {
    return static_cast<std::uint32_t>((c >> 3) * (ROWS * 128) + r * 128 + (((c & 7) ^ (r & 7)) << 4));
}

// One unit segment of a CTA's key-tile range: unit (kv head h, Q-tile pair
// qp) owns global key tiles [ustart, uend); the segment is [g0, g1).
struct Seg {
    int h, qp, ustart, uend, g0, g1;
};

// tab: the key-tile prefix over the Q-tile pairs (a.qp_tiles), copied to
// shared memory at kernel start when it fits: the binary search is a chain
// of dependent loads that every role runs at every segment switch (from
// global memory: ~1.5 us of L2 round trips on the critical path each time)
// (tab: 32-bit shared address of the copy, 0 = read a.qp_tiles)
__device__ __forceinline__ int tab_at(const PrefillArgs& a, std::uint32_t tab, int i) {
    if (!tab) return __ldg(a.qp_tiles + i);
    int v;
    asm volatile("ld.shared.s32 %0, [%1];\n" : "=r"(v) : "r"(tab + 4u * static_cast<std::uint32_t>(i)));
    return v;
}

__device__ __forceinline__ Seg seg_at(const PrefillArgs& a, std::uint32_t tab, int g, int g_end) {
    const int per_head = tab_at(a, tab, a.n_qp);
    Seg s;
    s.h = g / per_head;
    const int r = g - s.h * per_head;
    int lo = 0, hi = a.n_qp;  // largest qp with tab[qp] <= r
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (tab_at(a, tab, mid) <= r) lo = mid;
        else hi = mid;
    }
    s.qp = lo;
    s.ustart = s.h * per_head + tab_at(a, tab, lo);
    s.uend = s.h * per_head + tab_at(a, tab, lo + 1);
    s.g0 = g;
    s.g1 = min(s.uend, g_end);
    return s;
}

// Key tile (unit-local) that global position g of segment s computes. A unit
// cut across CTA ranges is shared by up to a few CTAs at the same time; ranked
// by (local time t = g - x * per_cta, CTA x), its positions take the unit's
// key tiles in ascending order, so every unit sweeps its keys from the start
// at the rate of the CTAs on it. The units of one kv head (the Q-tile pairs)
// then read nearby keys at any moment and each K/V tile is re-read from L2
// within a short window, instead of the cuts scattering the readers over the
// whole context (late 32K-key chunks: the kv heads' 134 MB of K/V do not fit
// the 126 MB L2). Online softmax and the part merge are order-free: only the
// causal mask needs the tile, and it takes it from here. Units inside one
// range keep the identity order.
// (per segment constants: the CTA range is x = range_id(), its local time is g - x * per_cta)
struct UnitOrder {
    int ustart, base, af, bl, nm, extra;  // base = x * per_cta; nm < 0: identity order
    __device__ __forceinline__ int tile(int g) const {
        if (nm < 0) return g - ustart;
        const int t = g - base;
        return max(0, t - af) + min(t, bl) + nm * t + (extra >= 0 ? extra + (t >= af ? 1 : 0) : 0);
    }
};

// The CTA's stream-K range index (blockIdx.x, or the interleaved order of
// PRISM_K4_PERM, which puts neighbouring ranges on CTAs launched apart)
__device__ __forceinline__ int range_id(const PrefillArgs& a) {
    const int b = static_cast<int>(blockIdx.x);
    if (!a.perm) return b;
    const int h = (static_cast<int>(gridDim.x) + 1) / 2;
    return (b & 1) ? h + (b >> 1) : (b >> 1);
}

__device__ __forceinline__ UnitOrder unit_order(const PrefillArgs& a, const Seg& s) {
    const int P = a.per_cta, x = range_id(a);
    const int f = s.ustart / P, l = (s.uend - 1) / P;
    UnitOrder o;
    o.ustart = s.ustart;
    o.base = x * P;
    o.af = s.ustart - f * P;  // CTA f holds local times [af, P) of the unit
    o.bl = s.uend - l * P;    // CTA l holds [0, bl)
    o.nm = f == l ? -1 : l - f - 1;  // CTAs whose whole range lies in the unit
    o.extra = x > f ? min(x, l) - f - 1 : -1;  // lower CTAs at the same local time (+ f if active)
    return o;
}

constexpr int kFastParts = 4;  // merges with at most this many parts take the latency-parallel path

template <int D, int G>
__global__ void __launch_bounds__(512, 1) k4_prefill(PrefillArgs a) {
    using S = PfShape<D>;
    extern __shared__ unsigned char smem_raw[];
    // 1024-byte aligned base (SW128 atoms), derived by pointer arithmetic on
    // the shared array so accesses through it stay LDS / STS
    unsigned char* smem = smem_raw + ((1024u - (saddr(smem_raw) & 1023u)) & 1023u);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    constexpr int kTQ = S::kM / G;  // query tokens per Q tile
    const int rid = range_id(a);
    const int g_begin = rid * a.per_cta;
    const int g_end = min(a.total, g_begin + a.per_cta);
    if (g_begin >= g_end) return;
    if (tid == 0) k4_cta_stamp(a.cta_trace, 0);
    const int n_kv = a.g.n_kv, n_q = n_kv * G;

    const std::uint32_t sQ = saddr(smem + S::kOffQ);
    const std::uint32_t sKV = saddr(smem + S::kOffKV);
    const std::uint32_t bar = saddr(smem + S::kOffBar);
    // q_full | q_empty | kv_full[H] | kv_empty[H] | s_full[2][2] | p_full[2][2] | pv_done[2][2] | o_free[2]
    // ([j][b]: Q tile j, tile parity b)
    const std::uint32_t b_qfull = bar, b_qempty = bar + 16, b_kvfull = bar + 32,
                        b_kvempty = b_kvfull + 8 * S::kHalves, b_sfull = b_kvempty + 8 * S::kHalves,
                        b_pfull = b_sfull + 32, b_pvdone = b_pfull + 32, b_ofree = b_pvdone + 32;
    std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(smem + S::kOffMisc);
    volatile int* merge_flag = reinterpret_cast<volatile int*>(smem + S::kOffMisc + 4);

    if (tid == 0) {
        for (int b = 0; b < 2; ++b) {
            mb_init(b_qfull + 8 * b, S::kLoaders);
            mb_init(b_qempty + 8 * b, 2);  // one commit per MMA issuer
        }
        for (int s = 0; s < S::kHalves; ++s) {
            mb_init(b_kvfull + 8 * s, S::kLoaders);
            mb_init(b_kvempty + 8 * s, 2);
        }
        for (int j = 0; j < 4; ++j) {
            mb_init(b_sfull + 8 * j, 1);
            mb_init(b_pfull + 8 * j, 128);
            mb_init(b_pvdone + 8 * j, 1);
        }
        for (int j = 0; j < 2; ++j) mb_init(b_ofree + 8 * j, 128);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    const bool tab_in_smem = a.tab_smem && a.n_qp + 1 <= S::kMaxTab;
    if (tab_in_smem) {
        std::int32_t* tab_s = reinterpret_cast<std::int32_t*>(smem + S::kOffTab);
        for (int i = tid; i <= a.n_qp; i += S::kThreads) tab_s[i] = __ldg(a.qp_tiles + i);
    }
    const std::uint32_t tab = tab_in_smem ? saddr(smem + S::kOffTab) : 0u;
    if (warp == 12) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(saddr(tmem_slot)),
                     "n"(S::kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const std::uint32_t tmem = *tmem_slot;
    // PDL (a chained launch of consecutive layers): the next K4 may launch
    // once every CTA of this one runs; its CTAs take the SMs this launch's
    // CTAs free and read q / K / V (never written by K4) at once. Global
    // writes (out, partials, tickets — the workspace and tickets are shared
    // by consecutive launches) wait for this launch's completion.
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    if (tid == 0 && a.cta_trace) {  // slot 1: the SM this CTA runs on
        unsigned sm;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
        a.cta_trace[blockIdx.x * 4 + 1] = sm;
    }
    // K half of local tile k is ring half 2k, its V half 2k + 1
    auto half_slot = [](int idx) { return idx % S::kHalves; };
    auto half_phase = [](int idx) { return static_cast<std::uint32_t>((idx / S::kHalves) & 1); };

    if (warp >= 8 && warp < 10) {
        // idle (registers only): the schedulers of the MMA warps (0, 1) carry
        // no loader, which measured +5% at 2K-token chunks
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(S::kRegsLoad));
    } else if (warp >= 10 && warp < 12) {
        // ------------------------------------------------------------ loaders
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(S::kRegsLoad));
        // Fixed rows per thread: lanes 2i and 2i+1 share a row (one 32-byte
        // sector per lane pair and instruction), lane parity h picks the odd
        // or even 16-byte chunks; loader warp w owns K/V tile rows 16w + i
        // and 32 + 16w + i (and rows 32m + 16w + i of the Q pair), so a thread
        // decodes its own rows' slot ids one tile ahead in registers and each
        // cp.async is one add + LDGSTS.
        const int w = warp - 10, h = lane & 1;
        const int ra = 16 * w + (lane >> 1), rb = ra + 32;  // ra & 7 == rb & 7
        constexpr int kCpl = D / 16;  // chunks per lane per row
        const char* base = reinterpret_cast<const char*>(a.g.base);
        const std::uint64_t v_delta = static_cast<std::uint64_t>(n_kv) * a.g.tpp * (D * 2);
        const int keys = a.first + a.chunk;  // the request's block-table row length
        std::uint32_t dsw_kv[kCpl], dsw_q[kCpl];  // swizzled chunk offsets within a row
#pragma unroll
        for (int i = 0; i < kCpl; ++i) {
            const int c = 2 * i + h;
            dsw_kv[i] = static_cast<std::uint32_t>((c >> 3) * (S::kN * 128) + (((c & 7) ^ (ra & 7)) << 4));
            dsw_q[i] = static_cast<std::uint32_t>((c >> 3) * (S::kM * 128) + (((c & 7) ^ (ra & 7)) << 4));
        }
        // src_bytes 0 (zero fill) reads nothing; q is a valid placeholder address
        const char* dummy = reinterpret_cast<const char*>(a.q);
        auto copy_row = [&](std::uint32_t dst_row, const std::uint32_t (&dsw)[kCpl], const char* src, bool ok) {
#if defined(K4_EXP) && (K4_EXP & 2)  // timing experiment: no K/V copies
            if (dst_row >= sKV) return;
#endif
            const char* p = (ok ? src : dummy) + h * 16;
            const int bytes = ok ? 16 : 0;
#pragma unroll
            for (int i = 0; i < kCpl; ++i) cp_async16_s(dst_row + dsw[i], p + i * 32, bytes);
        };
        auto load_sid = [&](int kt, int r) -> std::int32_t {
            const int key = kt * S::kN + r;
            return key < keys ? __ldg(a.row + key) : -1;
        };
        // byte offset of the row from the pool base, head block excluded; ~0: past the keys
        auto decode = [&](std::int32_t sid_raw) -> std::uint64_t {
            if (sid_raw < 0) return ~0ull;
            const std::uint32_t sid = static_cast<std::uint32_t>(sid_raw);
            const std::uint32_t page = slot_page(sid, a.g.magic);
            const std::uint32_t slot = sid - page * a.g.tpp;
            return static_cast<std::uint64_t>(page) * a.g.page_bytes + static_cast<std::uint64_t>(slot) * (D * 2);
        };
        // The loaders make their own copies visible to the tensor core: each
        // ring half is one cp.async group; kLag groups after issuing it, a
        // thread waits for it, fences the generic -> async proxy and arrives
        // on the half's full barrier (and on q_full for the group that also
        // carried the unit's Q pair), so the MMA warps only wait on barriers.
        // (a half of ring slot s is released once the MMA warps consumed it,
        // which needs only halves issued before it: kLag < kHalves suffices)
        constexpr int kLag = 2;
        static_assert(kLag < S::kHalves, "MMA progress must not need a half held back by the lag");
        int pend = 0, last_idx = -1;
        unsigned qbits = 0, qsel = 0;  // bit i: the group of half last_idx - i carried a Q pair, its buffer
        auto arrive_half = [&](int hidx, bool q, unsigned qb) {
            if (q) mb_arrive(b_qfull + 8 * qb);
            mb_arrive(b_kvfull + 8 * half_slot(hidx));
        };
        auto flush = [&]() {
            cp_async_wait<0>();
            fence_proxy_async();
            for (int i = pend - 1; i >= 0; --i) arrive_half(last_idx - i, (qbits >> i) & 1u, (qsel >> i) & 1u);
            pend = 0;
        };
        Seg la = seg_at(a, tab, g_begin, g_end);  // look-ahead cursor (tile g + 1)
        UnitOrder lo_ = unit_order(a, la);
        const int kt0 = lo_.tile(g_begin);
        std::uint64_t oa = decode(load_sid(kt0, ra)), ob = decode(load_sid(kt0, rb));
        int g = g_begin, s_idx = 0;
        while (g < g_end) {
            const Seg sg = seg_at(a, tab, g, g_end);
            // Q pair of the unit into buffer s_idx & 1 (the next segment's Q
            // loads while this one computes): rows of tile j = token (r / G) x
            // head (r % G), padding rows zero; committed with the segment's
            // first K half
            const unsigned qb = static_cast<unsigned>(s_idx & 1);
            if (s_idx > 1) {
                flush();  // the MMA warps need every issued half to release that buffer
                mb_wait(b_qempty + 8 * qb, ((s_idx - 2) >> 1) & 1);
            }
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                const int r = ra + 32 * m, j = r >> 7, rr = r & 127;
                const int tok = (2 * sg.qp + j) * kTQ + rr / G;
                const bool ok = rr < kTQ * G && tok < a.chunk;
                const char* src = reinterpret_cast<const char*>(
                    a.q + (static_cast<std::size_t>(ok ? tok : 0) * n_q + static_cast<std::size_t>(sg.h) * G + rr % G) * D);
                copy_row(sQ + (2 * qb + j) * S::kQB + rr * 128, dsw_q, src, ok);
            }
            if (lane == 0 && w == 0) k4_mark(a.dbg, 0, 1 + s_idx);  // loader: Q pair of segment issued
            const std::uint64_t kb = static_cast<std::uint64_t>(a.layer * 2 * n_kv + sg.h) * a.g.tpp * (D * 2);
            for (; g < sg.g1; ++g) {
                const int k = g - g_begin;
                std::int32_t na = -1, nb = -1;
                if (g + 1 < g_end) {
                    if (g + 1 >= la.g1) {
                        la = seg_at(a, tab, g + 1, g_end);
                        lo_ = unit_order(a, la);
                    }
                    const int kt = lo_.tile(g + 1);
                    na = load_sid(kt, ra);
                    nb = load_sid(kt, rb);
                }
#pragma unroll
                for (int kv = 0; kv < 2; ++kv) {
                    const int idx = 2 * k + kv;
                    const int hs = half_slot(idx);
                    if (idx >= S::kHalves) mb_wait(b_kvempty + 8 * hs, half_phase(idx) ^ 1u);
                    const char* blk = base + kb + (kv ? v_delta : 0);
                    copy_row(sKV + hs * S::kHalfB + ra * 128, dsw_kv, blk + oa, oa != ~0ull);
                    copy_row(sKV + hs * S::kHalfB + rb * 128, dsw_kv, blk + ob, ob != ~0ull);
                    cp_async_commit();
                    last_idx = idx;
                    qbits = (qbits << 1) | ((kv == 0 && g == sg.g0) ? 1u : 0u);
                    qsel = (qsel << 1) | qb;
                    if (++pend > kLag) {
                        cp_async_wait<kLag>();
                        fence_proxy_async();
                        arrive_half(idx - kLag, (qbits >> kLag) & 1u, (qsel >> kLag) & 1u);
                        --pend;
                    }
                }
                if (lane == 0 && w == 0) {
                    k4_stamp(a.trace, a.trace_cta, 0, k);
                    k4_mark(a.dbg, 1, 100 + k);  // loader: tile issued
                }
                oa = decode(na);
                ob = decode(nb);
            }
            ++s_idx;
        }
        flush();
    } else if (warp >= 12) {
        // ------------------------------------------------------------ MMA issue (warp 12)
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(S::kRegsLoad));
        // Warp 12 + j issues every MMA of Q tile j (the two Q tiles' pipelines
        // share only the K/V ring, whose slots are released by one commit of
        // each issuer). The whole warp runs the issue loop (uniform control
        // flow); one elected lane issues each tcgen05 op.
        if (warp < 14) {
            const int j = warp - 12;
            constexpr std::uint32_t idesc_s = f16_idesc(S::kM, S::kN, 0);
            constexpr std::uint32_t idesc_o = f16_idesc(S::kM, D, 1);
            const int n = g_end - g_begin;
            auto wait_half = [&](int idx) {
                mb_wait(b_kvfull + 8 * half_slot(idx), half_phase(idx));  // the loaders fenced the proxy
                tc_fence_after();
            };
            const std::uint32_t s_col = tmem + j * 2 * S::kN, o_col = tmem + S::kColO + j * D;
            // S_j(k) = Q_j · K(k)ᵀ into S buffer (j, k & 1): two tiles ahead of P_j·V
            Seg sc = seg_at(a, tab, g_begin, g_end);
            int sc_idx = 0;
            auto issue_s = [&](int k) {
                const int g = g_begin + k;
                if (g >= sc.g1) {  // a new unit segment: its Q pair
                    sc = seg_at(a, tab, g, g_end);
                    ++sc_idx;
                }
                const unsigned qb = static_cast<unsigned>(sc_idx & 1);
                if (g == sc.g0) mb_wait(b_qfull + 8 * qb, (sc_idx >> 1) & 1);
                const std::uint32_t dq = desc_lo(sQ + (2 * qb + j) * S::kQB, 16);
                if (j == 0 && lane == 0) k4_stamp(a.trace, a.trace_cta, 11, k);
                wait_half(2 * k);
                if (j == 0 && lane == 0) k4_stamp(a.trace, a.trace_cta, 12, k);
                const std::uint32_t dk = desc_lo(sKV + half_slot(2 * k) * S::kHalfB, 16);
                static_assert(S::kM * 128 / 16 == 1024 && S::kN * 128 / 16 == 512, "descriptor steps in tc_mma_s_tile");
                tc_mma_s_tile<D>(s_col + (k & 1) * S::kN, desc_of(dq), desc_of(dk), idesc_s);
                tc_commit_e(b_sfull + 8 * (2 * j + (k & 1)));
                tc_commit_e(b_kvempty + 8 * half_slot(2 * k));
                if (g + 1 == sc.g1) tc_commit_e(b_qempty + 8 * qb);  // last S of the segment: its Q buffer is free
                if (lane == 0) {
                    if (j == 0) k4_stamp(a.trace, a.trace_cta, 1, k);
                    k4_mark(a.dbg, 2 + j, 100 + k);  // MMA warp j: S(k) issued
                }
            };
            issue_s(0);
            if (n > 1) issue_s(1);
            Seg pc = seg_at(a, tab, g_begin, g_end);
            int pc_idx = 0;
            for (int k = 0; k < n; ++k) {
                const int g = g_begin + k;
                if (g >= pc.g1) {
                    pc = seg_at(a, tab, g, g_end);
                    ++pc_idx;
                }
                const bool fresh = g == pc.g0;
                // O_j (+)= P_j(k) · V(k), P_j in S buffer (j, k & 1)
                if (j == 0 && lane == 0) k4_stamp(a.trace, a.trace_cta, 8, k);
                mb_wait(b_pfull + 8 * (2 * j + (k & 1)), (k >> 1) & 1);
                if (fresh && pc_idx > 0) mb_wait(b_ofree + 8 * j, (pc_idx - 1) & 1);
                if (j == 0 && lane == 0) k4_stamp(a.trace, a.trace_cta, 9, k);
                wait_half(2 * k + 1);
                if (j == 0 && lane == 0) k4_stamp(a.trace, a.trace_cta, 10, k);
                const std::uint32_t dv = desc_lo(sKV + half_slot(2 * k + 1) * S::kHalfB, S::kN * 128);
                static_assert(S::kN == 64, "four K=16 steps in tc_mma_pv_tile");
                tc_mma_pv_tile(o_col, s_col + (k & 1) * S::kN, desc_of(dv), idesc_o, fresh ? 0u : 1u);
                tc_commit_e(b_pvdone + 8 * (2 * j + (k & 1)));
                tc_commit_e(b_kvempty + 8 * half_slot(2 * k + 1));
                if (lane == 0) {
                    k4_stamp(a.trace, a.trace_cta, j == 0 ? 2 : 7, k);
                    if (j == 0) k4_mark(a.dbg, 4, 100 + k);  // MMA warp 0: P·V(k) issued
                }
                if (k + 2 < n) issue_s(k + 2);
            }
        }
        __syncwarp();
    } else {
        // ------------------------------------------------------------ softmax warpgroups
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(S::kRegsSoftmax));
        const int j = warp >> 2;  // Q tile of the unit
        const int r = tid & 127;  // row = TMEM lane
        const std::uint32_t lane_base = static_cast<std::uint32_t>((warp & 3) * 32) << 16;
        const std::uint32_t tO = tmem + lane_base + S::kColO + j * D;
        const int tq = r / G;
        const int row = j * S::kM + r;  // row of the unit (partials)
        // Merge of a cut unit by the last of its parts to publish: every
        // part's (m, l, O / l) from the workspace, combined into `out`.
        auto merge_unit = [&](const Seg& ps) {
            const int first_cta = ps.ustart / a.per_cta, last_cta = (ps.uend - 1) / a.per_cta;
            const int parts = last_cta - first_cta + 1;
            const int tok = (2 * ps.qp + j) * kTQ + tq;
            const bool row_ok = r < kTQ * G && tok < a.chunk;
            __nv_bfloat16* dst =
                row_ok ? a.out + (static_cast<std::size_t>(tok) * n_q + static_cast<std::size_t>(ps.h) * G + r % G) * D
                       : nullptr;
            if (a.merge_fast && parts <= kFastParts) {
                __threadfence();
                // Latency-parallel combination (the usual case: a unit
                // cut into 2-4 parts): every part's (m, l) in one round of
                // loads, then per 32-column group all parts' O rows at
                // once — 1 + D / 32 dependent L2 round trips instead of
                // (2 + D / 32) x parts.
                auto slot_of = [&](int cta) { return 2 * cta + (cta * a.per_cta >= ps.ustart ? 0 : 1); };
                int sl[kFastParts];
                float2 ml[kFastParts];
#pragma unroll
                for (int t = 0; t < kFastParts; ++t) {
                    sl[t] = slot_of(min(first_cta + t, last_cta));
                    if (t < parts) ml[t] = __ldcg(a.part_ml + static_cast<std::size_t>(sl[t]) * 256 + row);
                }
                float mm = -INFINITY;
#pragma unroll
                for (int t = 0; t < kFastParts; ++t)
                    if (t < parts) mm = fmaxf(mm, ml[t].x);
                float ll = 0.f;
#pragma unroll
                for (int t = 0; t < kFastParts; ++t)
                    if (t < parts) ll += ml[t].x == -INFINITY ? 0.f : ml[t].y * fast_exp2(ml[t].x - mm);
                const float inv = ll > 0.f ? 1.f / ll : 0.f;
                float wt[kFastParts];
#pragma unroll
                for (int t = 0; t < kFastParts; ++t)
                    wt[t] = (t < parts && ml[t].x != -INFINITY) ? fast_exp2(ml[t].x - mm) * ml[t].y * inv : 0.f;
#pragma unroll 1
                for (int cg = 0; cg < D / 32; ++cg) {
                    uint2 h[kFastParts][8];
#pragma unroll
                    for (int t = 0; t < kFastParts; ++t)
#pragma unroll
                        for (int q = 0; q < 8; ++q)
                            h[t][q] = t < parts ? __ldcg(a.part_o + (static_cast<std::size_t>(sl[t]) * (D / 4) +
                                                                     cg * 8 + q) * 256 + row)
                                                : make_uint2(0u, 0u);
                    float4 acc[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                        for (int t = 0; t < kFastParts; ++t) {
                            const float2 lo = unpack_f16(h[t][q].x), hi = unpack_f16(h[t][q].y);
                            acc[q].x += wt[t] * lo.x;
                            acc[q].y += wt[t] * lo.y;
                            acc[q].z += wt[t] * hi.x;
                            acc[q].w += wt[t] * hi.y;
                        }
                    }
                    if (row_ok) {
#pragma unroll
                        for (int q = 0; q < 8; q += 2) {
                            *reinterpret_cast<uint4*>(dst + cg * 32 + 4 * q) =
                                make_uint4(pack_bf16(acc[q].x, acc[q].y), pack_bf16(acc[q].z, acc[q].w),
                                           pack_bf16(acc[q + 1].x, acc[q + 1].y),
                                           pack_bf16(acc[q + 1].z, acc[q + 1].w));
                        }
                    }
                }
            } else {
                __threadfence();
                // online combination of the parts' (m, l, O) rows
                auto slot_of = [&](int cta) { return 2 * cta + (cta * a.per_cta >= ps.ustart ? 0 : 1); };
                float mm = -INFINITY;
                for (int cta = first_cta; cta <= last_cta; ++cta)
                    mm = fmaxf(mm, __ldcg(a.part_ml + static_cast<std::size_t>(slot_of(cta)) * 256 + row).x);
                float ll = 0.f;
                for (int cta = first_cta; cta <= last_cta; ++cta) {
                    const float2 ml = __ldcg(a.part_ml + static_cast<std::size_t>(slot_of(cta)) * 256 + row);
                    ll += ml.x == -INFINITY ? 0.f : ml.y * fast_exp2(ml.x - mm);
                }
                const float inv = ll > 0.f ? 1.f / ll : 0.f;
#pragma unroll 1
                for (int cg = 0; cg < D / 32; ++cg) {
                    float4 acc[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
                    for (int cta = first_cta; cta <= last_cta; ++cta) {
                        const int sl = slot_of(cta);
                        const float2 pml = __ldcg(a.part_ml + static_cast<std::size_t>(sl) * 256 + row);
                        // the partial is O / l: weight by l
                        const float wt = pml.x == -INFINITY ? 0.f : fast_exp2(pml.x - mm) * pml.y * inv;
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            const uint2 h4 =
                                __ldcg(a.part_o + (static_cast<std::size_t>(sl) * (D / 4) + cg * 8 + q) * 256 + row);
                            const float2 lo = unpack_f16(h4.x), hi = unpack_f16(h4.y);
                            acc[q].x += wt * lo.x;
                            acc[q].y += wt * lo.y;
                            acc[q].z += wt * hi.x;
                            acc[q].w += wt * hi.y;
                        }
                    }
                    if (row_ok) {
#pragma unroll
                        for (int q = 0; q < 8; q += 2) {
                            *reinterpret_cast<uint4*>(dst + cg * 32 + 4 * q) =
                                make_uint4(pack_bf16(acc[q].x, acc[q].y), pack_bf16(acc[q].z, acc[q].w),
                                           pack_bf16(acc[q + 1].x, acc[q + 1].y),
                                           pack_bf16(acc[q + 1].z, acc[q + 1].w));
                        }
                    }
                }
            }
        };
        // a mid-range cut unit whose ticket was taken early (release atomic,
        // result checked at the range's next epilogue)
        bool pend = false;
        int pend_old = 0;
        Seg pend_seg{};
        int k = 0, g = g_begin;
        bool pdl_waited = false;
        // PV_j(k) completes phase k >> 1 of pv_done[j][k & 1]. Whenever this
        // warpgroup waits for PV_j(k) (k = its current tile - 1 or its last
        // tile), PV_j(k-2) is complete (it was issued before S_j(k), and MMAs
        // and their commits complete in issue order) and PV_j(k+2) cannot
        // be issued yet (it needs this warpgroup's P_j(k+2)): the parity
        // wait is exact.
        auto wait_pv = [&](int kk) {
            mb_wait(b_pvdone + 8 * (2 * j + (kk & 1)), (kk >> 1) & 1);
            tc_fence_after();
        };
        while (g < g_end) {
            const Seg sg = seg_at(a, tab, g, g_end);
            const UnitOrder ord = unit_order(a, sg);
            const int tok = (2 * sg.qp + j) * kTQ + tq;
            const bool row_ok = r < kTQ * G && tok < a.chunk;
            const int pos = row_ok ? a.first + tok : -1;  // last key this row may attend
            float m_run = -INFINITY, l_run = 0.f;
            for (; g < sg.g1; ++g, ++k) {
                const int b = k & 1;
                mb_wait(b_sfull + 8 * (2 * j + b), (k >> 1) & 1);
                tc_fence_after();
                if (r == 0) {
                    k4_stamp(a.trace, a.trace_cta, j == 0 ? 3 : 5, k);
                    if (j == 0) k4_mark(a.dbg, 5, 100 + k);  // softmax 0: has S(k)
                }
#if defined(K4_EXP) && (K4_EXP & 1)  // timing experiment: no softmax
                if (true) {
                    tc_fence_before();
                    mb_arrive(b_pfull + 8 * (2 * j + b));
                    continue;
                }
#endif
                const std::uint32_t tS = tmem + lane_base + j * 2 * S::kN + b * S::kN;
                const int k0 = ord.tile(g) * S::kN;
                // the tile's S row in registers (one tcgen05.ld wait), row max
                // with 8 independent partial maxima; tiles entirely below the
                // diagonal skip the causal mask
                const bool full = k0 + S::kN - 1 <= pos;
                const int lim = pos - k0;  // last visible column of this tile
                static_assert(S::kN == 64, "one x64 TMEM load per S row");
                float v[S::kN];
                tc_ld64(tS, v);
                if (!full) {
#pragma unroll
                    for (int q = 0; q < S::kN; ++q) v[q] = q <= lim ? v[q] : -INFINITY;
                }
                float mx[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) mx[q] = v[q];
#pragma unroll
                for (int q = 8; q < S::kN; ++q) mx[q & 7] = fmaxf(mx[q & 7], v[q]);
                float mt = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                                 fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
                mt *= a.scale_log2;  // scale > 0: max commutes with the scaling
                bool rescale = false;
                float alpha = 1.f;
                if (mt > m_run + a.rescale_thr) {
                    if (m_run != -INFINITY) {
                        alpha = fast_exp2(m_run - mt);
                        rescale = true;
                    }
                    m_run = mt;
                    l_run *= alpha;
                }
                const float m_use = m_run == -INFINITY ? 0.f : m_run;
                // O_j *= alpha for the rows whose max moved (warp-collective
                // TMEM access; rare with the 2^8 threshold): PV_j(k-1) must be
                // complete (never needed on a unit's first tile: m was -inf)
                if (__any_sync(0xffffffffu, rescale)) {
                    wait_pv(k - 1);
#pragma unroll
                    for (int cc = 0; cc < D / 32; ++cc) {
                        float o[32];
                        tc_ld32(tO + cc * 32, o);
#pragma unroll
                        for (int q = 0; q < 32; ++q) o[q] *= alpha;
                        tc_st32(tO + cc * 32, o);
                    }
                }
                // p = exp2(s - m) (masked s = -inf -> 0), row sum, bf16 P over
                // the buffer's first columns (the S row is already in registers)
                // packed fp32x2 arithmetic (FFMA2 / FADD2) around the MUFU ex2
                // (a polynomial exp2 on the FMA pipe for part of the pairs was
                // measured: no gain, the MMA issue path bounds the tile rate)
                const float2 sc2 = make_float2(a.scale_log2, a.scale_log2), nm2 = make_float2(-m_use, -m_use);
                float2 ls[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) ls[q] = make_float2(0.f, 0.f);
                std::uint32_t pk[S::kN / 2];
#pragma unroll
                for (int i = 0; i < S::kN / 2; ++i) {
                    const float2 x = __ffma2_rn(make_float2(v[2 * i], v[2 * i + 1]), sc2, nm2);
                    const float2 pr = make_float2(fast_exp2(x.x), fast_exp2(x.y));
                    ls[i & 3] = __fadd2_rn(ls[i & 3], pr);
                    pk[i] = pack_bf16(pr.x, pr.y);
                }
                tc_st32_nowait(tS, pk);
                asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
                const float2 l2 = __fadd2_rn(__fadd2_rn(ls[0], ls[1]), __fadd2_rn(ls[2], ls[3]));
                l_run += l2.x + l2.y;
                tc_fence_before();
                mb_arrive(b_pfull + 8 * (2 * j + b));
                if (r == 0) {
                    k4_stamp(a.trace, a.trace_cta, j == 0 ? 4 : 6, k);
                    if (j == 0) k4_mark(a.dbg, 6, 100 + k);  // softmax 0: posted P(k)
                }
            }
            // ---- epilogue of the unit segment: O_j complete after PV_j(last)
            wait_pv(k - 1);
            if (j == 0 && r == 0) k4_mark(a.dbg, 7, 100 + k);  // softmax 0: epilogue
            if (!pdl_waited) {  // first global write of this thread (see launch_dependents)
                asm volatile("griddepcontrol.wait;\n" ::: "memory");
                pdl_waited = true;
                if (tid == 0) k4_cta_stamp(a.cta_trace, 2);
            }
            if (pend) {
                if (tid == 0) {
                    const int pu = pend_seg.h * a.n_qp + pend_seg.qp;
                    const int pparts = (pend_seg.uend - 1) / a.per_cta - pend_seg.ustart / a.per_cta + 1;
                    const int last = pend_old == pparts - 1;
                    if (last) {
                        __threadfence();  // acquire side: the other parts' partials
                        a.tickets[pu] = 0;
                    }
                    *merge_flag = last;
                }
                asm volatile("bar.sync 1, 256;\n" ::: "memory");
                if (*merge_flag) merge_unit(pend_seg);
                asm volatile("bar.sync 1, 256;\n" ::: "memory");  // merge_flag is rewritten below
                pend = false;
            }
            const int u = sg.h * a.n_qp + sg.qp;
            if (r == 0 && j == 0) k4_stamp(a.trace, a.trace_cta, 13, k - 1);  // epilogue: O complete
            const int first_cta = sg.ustart / a.per_cta, last_cta = (sg.uend - 1) / a.per_cta;
            const int parts = last_cta - first_cta + 1;
            __nv_bfloat16* dst =
                row_ok ? a.out + (static_cast<std::size_t>(tok) * n_q + static_cast<std::size_t>(sg.h) * G + r % G) * D
                       : nullptr;
            if (parts == 1) {
                const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
#pragma unroll
                for (int cc = 0; cc < D / 32; ++cc) {
                    float o[32];
                    tc_ld32(tO + cc * 32, o);
                    if (row_ok) {
#pragma unroll
                        for (int q = 0; q < 32; q += 8) {
                            *reinterpret_cast<uint4*>(dst + cc * 32 + q) =
                                make_uint4(pack_bf16(o[q] * inv, o[q + 1] * inv), pack_bf16(o[q + 2] * inv, o[q + 3] * inv),
                                           pack_bf16(o[q + 4] * inv, o[q + 5] * inv),
                                           pack_bf16(o[q + 6] * inv, o[q + 7] * inv));
                        }
                    }
                }
                tc_fence_before();
                mb_arrive(b_ofree + 8 * j);
            } else {
                // publish this CTA's partial of the unit (slot 2c: the range's
                // first segment, 2c + 1: its last), then the last publisher merges
                const int slot = 2 * rid + (sg.g0 == g_begin ? 0 : 1);
                // O / l: |values| <= max |V|, so fp16 keeps 2^-11 relative
                // precision in half the bytes of an fp32 partial
                const float inv_l = l_run > 0.f ? 1.f / l_run : 0.f;
#pragma unroll
                for (int cc = 0; cc < D / 32; ++cc) {
                    float o[32];
                    tc_ld32(tO + cc * 32, o);
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        a.part_o[(static_cast<std::size_t>(slot) * (D / 4) + cc * 8 + q) * 256 + row] =
                            make_uint2(pack_f16(o[4 * q] * inv_l, o[4 * q + 1] * inv_l),
                                       pack_f16(o[4 * q + 2] * inv_l, o[4 * q + 3] * inv_l));
                }
                a.part_ml[static_cast<std::size_t>(slot) * 256 + row] = make_float2(m_run, l_run);
                tc_fence_before();
                mb_arrive(b_ofree + 8 * j);
                // the barrier orders every thread's partial stores before
                // thread 0's gpu-scope release (fence + ticket), which is
                // cumulative over them (the usual semaphore pattern)
                if (r == 0 && j == 0) k4_stamp(a.trace, a.trace_cta, 14, k - 1);  // partial stored
                asm volatile("bar.sync 1, 256;\n" ::: "memory");
                if (sg.g1 < g_end && a.early_ticket) {
                    // more of this range follows: thread 0 takes the ticket with
                    // a release atomic (cumulative over the barrier) and nobody
                    // waits for its result here; the range's next epilogue
                    // checks it and merges the unit if this part was the last
                    if (tid == 0) {
                        asm volatile("atom.add.release.gpu.global.s32 %0, [%1], 1;\n"
                                     : "=r"(pend_old) : "l"(a.tickets + u) : "memory");
                    }
                    pend = true;
                    pend_seg = sg;
                    continue;
                }
                if (tid == 0) {
                    __threadfence();
                    const int prev = atomicAdd(a.tickets + u, 1);
                    const int last = prev == parts - 1;
                    if (last) a.tickets[u] = 0;  // no other CTA touches it again in this launch
                    __threadfence();
                    *merge_flag = last;
                }
                asm volatile("bar.sync 1, 256;\n" ::: "memory");
                if (r == 0 && j == 0) k4_stamp(a.trace, a.trace_cta, 15, k - 1);  // ticket taken
                if (*merge_flag) merge_unit(sg);
            }
        }
        tc_fence_before();
    }
    __syncthreads();
    if (tid == 0) k4_cta_stamp(a.cta_trace, 3);
    if (warp == 12) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(S::kTmemCols)
                     : "memory");
    }
}

template <int D, int G>
void launch_pf(const PrefillArgs& a, int grid, cudaStream_t stream, bool chained) {
    using S = PfShape<D>;
    static bool init = false;
    if (!init) {
        PRISM_CUDA(cudaFuncSetAttribute(k4_prefill<D, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, S::kSmem));
        init = true;
    }
    // chained: a programmatic dependent of the previous K4 launch on this
    // stream (its CTAs start on the SMs the previous launch's CTAs free, and
    // wait for it only before their first global write)
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(grid));
    cfg.blockDim = dim3(S::kThreads);
    cfg.dynamicSmemBytes = S::kSmem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = chained ? 1 : 0;
    PRISM_CUDA(cudaLaunchKernelEx(&cfg, k4_prefill<D, G>, a));
    PRISM_CUDA(cudaGetLastError());
}

template <int D>
void launch_pf_d(int group, const PrefillArgs& a, int grid, cudaStream_t stream, bool chained) {
    switch (group) {
        case 1: launch_pf<D, 1>(a, grid, stream, chained); break;
        case 2: launch_pf<D, 2>(a, grid, stream, chained); break;
        case 3: launch_pf<D, 3>(a, grid, stream, chained); break;
        case 4: launch_pf<D, 4>(a, grid, stream, chained); break;
        case 5: launch_pf<D, 5>(a, grid, stream, chained); break;
        case 6: launch_pf<D, 6>(a, grid, stream, chained); break;
        case 7: launch_pf<D, 7>(a, grid, stream, chained); break;
        case 8: launch_pf<D, 8>(a, grid, stream, chained); break;
        default: throw std::runtime_error("prefill_attention: unsupported GQA group");
    }
}

}  // namespace

static unsigned* g_k4_dbg_host = nullptr;
static unsigned* k4_debug_words() {
    static unsigned* dev = [] {
        if (!std::getenv("PRISM_K4_DEBUG")) return static_cast<unsigned*>(nullptr);
        PRISM_CUDA(cudaHostAlloc(&g_k4_dbg_host, 64 * sizeof(unsigned), cudaHostAllocMapped));
        std::memset(g_k4_dbg_host, 0, 64 * sizeof(unsigned));
        unsigned* p = nullptr;
        PRISM_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&p), g_k4_dbg_host, 0));
        return p;
    }();
    return dev;
}

// Progress words of the last K4 launch's CTA 0 (PRISM_K4_DEBUG), readable
// while the kernel runs; 0 words when debugging is off.
static unsigned long long* k4_trace_buf() {
    static unsigned long long* dev = [] {
        if (!std::getenv("PRISM_K4_TRACE") && !std::getenv("PRISM_K4_CTA_TRACE"))
            return static_cast<unsigned long long*>(nullptr);
        unsigned long long* p = nullptr;
        PRISM_CUDA(cudaMalloc(&p, 16 * 1024 * sizeof(unsigned long long)));
        PRISM_CUDA(cudaMemset(p, 0, 16 * 1024 * sizeof(unsigned long long)));
        return p;
    }();
    return dev;
}

// Timeline of the last traced K4 launch (synchronous copy); 0 when off.
int k4_trace_read(unsigned long long* out, int n) {
    unsigned long long* d = k4_trace_buf();
    if (!d) return 0;
    const int m = n < 16 * 1024 ? n : 16 * 1024;
    PRISM_CUDA(cudaDeviceSynchronize());
    PRISM_CUDA(cudaMemcpy(out, d, m * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    return m;
}

int k4_debug_read(unsigned* out, int n) {
    if (!g_k4_dbg_host) return 0;
    const int m = n < 64 ? n : 64;
    for (int i = 0; i < m; ++i) out[i] = reinterpret_cast<volatile unsigned*>(g_k4_dbg_host)[i];
    return m;
}

// Host side of the launch, shared by the engine path (EngineDeviceImpl) and
// the pool-level op (PagedCtx): the key-tile prefix over the Q-tile pairs
// depends only on (first, chunk), so it is uploaded once per chunk, not per
// layer; the stream-K cut uses one CTA per SM.
template <class Ctx>
void launch_k4(Ctx& d, PrefillArgs a) {
    constexpr int kN = 64;
    static const int sms = [] {
        int dev = 0, n = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (const char* e = std::getenv("PRISM_K4_SMS")) n = std::max(1, std::min(n, std::atoi(e)));  // experiments
        return n;
    }();
    // PDL only behind this engine's own K4 (PRISM_K4_PDL=0 disables)
    static const bool pdl = [] {
        const char* e = std::getenv("PRISM_K4_PDL");
        return !(e && e[0] == '0');
    }();
    bool chained = pdl && d.k4_chain;
    const int tq = 128 / d.group;
    const int n_qp = ((a.chunk + tq - 1) / tq + 1) / 2;
    if (d.pf_first != a.first || d.pf_chunk != a.chunk) {
        chained = false;  // the prefix upload below precedes this launch
        d.pf_prefix.ensure(static_cast<std::size_t>(n_qp) + 1);
        std::int32_t acc = 0;
        for (int qp = 0; qp < n_qp; ++qp) {
            d.pf_prefix.host[qp] = acc;
            const int kv_len = a.first + std::min(a.chunk, (2 * qp + 2) * tq);
            acc += (kv_len + kN - 1) / kN;
        }
        d.pf_prefix.host[n_qp] = acc;
        d.pf_prefix.upload(static_cast<std::size_t>(n_qp) + 1, d.stream);
        d.pf_first = a.first;
        d.pf_chunk = a.chunk;
        d.pf_per_head = acc;
    }
    a.n_qp = n_qp;
    a.qp_tiles = d.pf_prefix.dev;
    a.total = d.n_kv * d.pf_per_head;
    // one CTA per SM; a small launch (a short prefill chunk) spreads its
    // tiles over as many CTAs as there are tiles (latency, not throughput)
    a.per_cta = std::max(1, (a.total + sms - 1) / sms);
    const int grid = (a.total + a.per_cta - 1) / a.per_cta;
    const std::size_t slots = 2 * static_cast<std::size_t>(grid);
    float* ws = d.attn_workspace(slots * 256 * d.head_dim + slots * 256 * 2);
    a.part_o = reinterpret_cast<uint2*>(ws);
    a.part_ml = reinterpret_cast<float2*>(ws + slots * 256 * d.head_dim);
    a.tickets = d.attn_counters(static_cast<std::size_t>(d.n_kv) * n_qp);
    a.dbg = k4_debug_words();
    // PRISM_K4_TRACE: tile stamps of CTA 0 (rows 0-12 of the buffer);
    // PRISM_K4_CTA_TRACE: per-CTA timelines of 5 consecutive launches in
    // rows 13-15 ([launch % 5][CTA < 148][4])
    static const bool tile_trace = std::getenv("PRISM_K4_TRACE") != nullptr;
    static const bool cta_trace = std::getenv("PRISM_K4_CTA_TRACE") != nullptr;
    static unsigned long long cta_launch = 0;
    static const int trace_cta = [] {
        const char* e = std::getenv("PRISM_K4_TRACE_CTA");
        return e ? std::atoi(e) : 0;
    }();
    a.trace = tile_trace ? k4_trace_buf() : nullptr;
    a.trace_cta = trace_cta;
    a.cta_trace = (cta_trace && grid <= 148) ? k4_trace_buf() + 13 * 1024 + (cta_launch++ % 5) * 148 * 4 : nullptr;
    chained = chained && d.k4_chain;  // a workspace / counter reallocation breaks the chain
    if (d.head_dim == 128) {
        launch_pf_d<128>(d.group, a, grid, d.stream, chained);
    } else {
        launch_pf_d<64>(d.group, a, grid, d.stream, chained);
    }
    d.k3_chain = false;
    d.k4_chain = true;
}

int k4_early_ticket() {  // PRISM_K4_EARLY=0: every ticket taken and checked at once (A/B)
    static const int v = [] {
        const char* e = std::getenv("PRISM_K4_EARLY");
        return (e && e[0] == '0') ? 0 : 1;
    }();
    return v;
}

int k4_tab_smem() {  // PRISM_K4_TAB=0: seg_at reads the prefix from global memory (A/B)
    static const int v = [] {
        const char* e = std::getenv("PRISM_K4_TAB");
        return (e && e[0] == '0') ? 0 : 1;
    }();
    return v;
}

int k4_perm() {  // PRISM_K4_PERM=1: interleaved CTA -> range order (experiment)
    static const int v = [] {
        const char* e = std::getenv("PRISM_K4_PERM");
        return (e && e[0] == '1') ? 1 : 0;
    }();
    return v;
}

int k4_merge_fast() {  // PRISM_K4_MERGE=0: the per-part merge loop only (A/B)
    static const int v = [] {
        const char* e = std::getenv("PRISM_K4_MERGE");
        return (e && e[0] == '0') ? 0 : 1;
    }();
    return v;
}

void launch_prefill_attention(EngineDeviceImpl& d, int layer, const void* q, void* out, float scale) {
    if (layer < 0 || layer >= d.n_layers) throw std::runtime_error("prefill_attention: bad layer");
    if (d.prefill_chunk <= 0) return;
    if (d.head_dim != 64 && d.head_dim != 128) throw std::runtime_error("prefill_attention: head_dim must be 64 or 128");
    PrefillArgs a{};
    a.g = d.geom;
    a.layer = layer;
    a.q = static_cast<const __nv_bfloat16*>(q);
    a.out = static_cast<__nv_bfloat16*>(out);
    a.row = d.table + d.prefill_row;
    a.first = d.prefill_first;
    a.chunk = d.prefill_chunk;
    a.scale_log2 = scale * 1.4426950408889634f;
    static const float thr = [] {
        const char* e = std::getenv("PRISM_K4_RESCALE_THR");
        return e ? static_cast<float>(std::atof(e)) : 8.f;
    }();
    a.rescale_thr = thr;
    a.merge_fast = k4_merge_fast();
    a.perm = k4_perm();
    a.tab_smem = k4_tab_smem();
    a.early_ticket = k4_early_ticket();
    launch_k4(d, a);
}

void prefill_attention(msim::engine::Engine& eng, int layer, const void* q, void* out, float scale) {
    launch_prefill_attention(impl_of(eng), layer, q, out, scale);
}

void PagedCtx::prefill_attention(int layer, const std::int32_t* slot_ids, int first, int n_tokens, const void* q,
                                 void* out, float scale) {
    if (layer < 0 || layer >= n_layers) throw std::out_of_range("paged prefill_attention: bad layer");
    if (n_tokens <= 0) return;
    if (first < 0) throw std::invalid_argument("paged prefill_attention: first must be >= 0");
    if (!slot_ids || !q || !out) throw std::invalid_argument("paged prefill_attention: null pointer");
    PRISM_CUDA(cudaSetDevice(vmm->ordinal()));
    PrefillArgs a{};
    a.g = geom;
    a.layer = layer;
    a.q = static_cast<const __nv_bfloat16*>(q);
    a.out = static_cast<__nv_bfloat16*>(out);
    a.row = slot_ids;
    a.first = first;
    a.chunk = n_tokens;
    a.scale_log2 = scale * 1.4426950408889634f;
    a.rescale_thr = 8.f;
    a.merge_fast = k4_merge_fast();
    a.perm = k4_perm();
    a.tab_smem = k4_tab_smem();
    a.early_ticket = k4_early_ticket();
    launch_k4(*this, a);
}

int last_step_prefill_tokens(const msim::engine::Engine& eng) { return impl_of(eng).prefill_chunk; }
int last_step_prefill_first(const msim::engine::Engine& eng) { return impl_of(eng).prefill_first; }
std::uint64_t last_step_prefill_request(const msim::engine::Engine& eng) { return impl_of(eng).prefill_request; }

}  // namespace prism
