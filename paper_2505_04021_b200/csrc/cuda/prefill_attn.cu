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
// One CTA = one (query tile, kv head) work item. The G q heads of a kv head
// are packed into the MMA's M dimension: row r = token (r / G) x head (r % G),
// 128 rows = floor(128 / G) tokens, so one K/V tile feeds all G heads.
// Warp roles (256 threads = 2 warps per SM sub-partition, so up to 255
// registers per thread; one CTA per SM):
//   warps 0-3  softmax / correction / epilogue: thread r owns row r = TMEM
//              lane r; reads S rows with tcgen05.ld, online softmax in the log2
//              domain with lazy rescaling (O in TMEM is rescaled only when a
//              row max grows by more than 2^8), writes P (bf16) to shared
//              memory, final O / l to global;
//   warps 4-6  loaders: gather the Q tile and each 64-key K/V tile from the
//              pages with cp.async (16 B per thread-op) into 128B-swizzled
//              K-major tiles (the UMMA canonical layout), 5-stage ring
//              (64-key tiles: a deep ring hides the gather latency);
//              cp.async.mbarrier.arrive signals a stage without blocking the
//              loader (the MMA thread fences the generic->async proxy);
//   warp 7     TMEM allocation, and one lane issues every tcgen05.mma:
//              S = Q·Kᵀ (M=128, N=64, K=head_dim) into one of two TMEM S
//              buffers, O += P·V (M=128, N=head_dim, K=64; V used MN-major)
//              into the TMEM O accumulator; completion reaches the other
//              roles through tcgen05.commit on mbarriers.
// S(t+1) is issued before P(t)·V(t), so the tensor core computes the next
// scores while the softmax warps work on the current ones; P is double
// buffered, so the softmax of tile t+1 overlaps P(t)·V(t) (only a rare O
// rescale waits for it).
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <stdexcept>

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
    unsigned long long* trace;  // PRISM_K4_TRACE: [5][1024] globaltimer stamps of CTA (0,0), else null
    unsigned* dbg;            // PRISM_K4_DEBUG: host-mapped progress words (CTA (0,0) only), else null
};

// timeline stamp (no-op unless PRISM_K4_TRACE): role 0 loader issued tile t,
// 1 S(t) issued, 2 P(t)·V(t) issued, 3 softmax has S(t), 4 softmax posted P(t)
__device__ __forceinline__ void k4_stamp(unsigned long long* tr, int role, int t) {
    if (tr && blockIdx.x == 0 && blockIdx.y == 0 && t < 1024) {
        unsigned long long ns;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
        tr[role * 1024 + t] = ns;
    }
}

// progress marker for hang diagnosis (no-op unless PRISM_K4_DEBUG)
__device__ __forceinline__ void k4_mark(unsigned* dbg, int slot, unsigned v) {
    if (dbg && blockIdx.x == 0 && blockIdx.y == 0) {
        *reinterpret_cast<volatile unsigned*>(dbg + slot) = v;
        __threadfence_system();
    }
}

template <int D>
struct PfShape {
    static constexpr int kM = 128;            // MMA rows (packed token x head)
    static constexpr int kN = 128;            // keys per K/V tile
    static constexpr int kStages = 3;         // K/V ring depth
    static constexpr int kSub = D / 64;       // 64-element (128 B) swizzle atoms along head_dim
    static constexpr int kQB = kM * D * 2;    // Q tile bytes
    static constexpr int kKB = kN * D * 2;    // K (or V) tile bytes
    static constexpr int kStageB = 2 * kKB;   // K + V
    static constexpr int kOffQ = 0;
    static constexpr int kOffKV = kOffQ + kQB;
    static constexpr int kOffRows = kOffKV + kStages * kStageB;  // [2][kN] K row offsets / 128 B (loaders)
    static constexpr int kOffBar = kOffRows + 2 * kN * 4;
    static constexpr int kBars = 2 * kStages + 8;
    static constexpr int kSmem = kOffBar + kBars * 8 + 16 + 1024;  // + TMEM address slot + alignment slack
    static constexpr int kThreads = 256;
    static constexpr int kLoaders = 96;   // warps 4-6
    static constexpr std::uint32_t kTmemCols = 512;  // S0 [0,128) S1 [128,256) O [256, 256+D)
    // TMEM columns: S(t & 1) [kN each] | P(t & 1) [kN / 2 each: bf16 pairs] | O [D]
    static constexpr std::uint32_t kColP = 2 * kN;
    static constexpr std::uint32_t kColO = kColP + kN;
};

// ---------------------------------------------------------------- PTX helpers
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
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_commit(std::uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(bar)
                 : "memory");
}
// D[tmem] (+)= A[smem] · B[smem], kind::f16 (bf16 in, fp32 accumulate)
__device__ __forceinline__ void tc_mma(std::uint32_t d_tmem, std::uint64_t a_desc, std::uint64_t b_desc,
                                       std::uint32_t idesc, std::uint32_t accumulate) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
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

// D[tmem] (+)= A[tmem] · B[smem]: the A operand (P) read from tensor memory,
// lane = row, two bf16 K-elements per 32-bit column (8 columns per K=16 step)
__device__ __forceinline__ void tc_mma_ts(std::uint32_t d_tmem, std::uint32_t a_tmem, std::uint64_t b_desc,
                                          std::uint32_t idesc, std::uint32_t accumulate) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// 16 consecutive 32-bit columns of this thread's TMEM lane (no wait)
__device__ __forceinline__ void tc_st16_nowait(std::uint32_t taddr, const std::uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
        "%14, %15, %16};\n" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
        "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
}

// Shared-memory matrix descriptor (sm_100 "version 1"), 128-byte swizzle.
// K-major canonical layout ((8,m),(T,2)):((8T,SBO),(1,T)): rows of 128 B,
// 8-row groups 1024 B apart (SBO), LBO unused (1). MN-major canonical layout
// ((T,8,n),(8,k)):((1,T,LBO),(8T,SBO)): 64-element atoms along MN `lbo` bytes
// apart, 8-row K groups 1024 B apart.
__device__ __forceinline__ std::uint64_t sw128_desc(std::uint32_t addr, std::uint32_t lbo_bytes) {
    std::uint64_t d = 0;
    d |= static_cast<std::uint64_t>((addr >> 4) & 0x3fff);
    d |= static_cast<std::uint64_t>((lbo_bytes >> 4) & 0x3fff) << 16;
    d |= static_cast<std::uint64_t>((1024u >> 4) & 0x3fff) << 32;
    d |= static_cast<std::uint64_t>(1) << 46;  // version (sm_100)
    d |= static_cast<std::uint64_t>(2) << 61;  // SWIZZLE_128B
    return d;
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

template <int D, int G>
__global__ void __launch_bounds__(256, 1) k4_prefill(PrefillArgs a) {
    using S = PfShape<D>;
    extern __shared__ unsigned char smem_raw[];
    // 1024-byte aligned base (SW128 atoms), derived by pointer arithmetic on
    // the shared array so accesses through it stay LDS / STS
    unsigned char* smem = smem_raw + ((1024u - (saddr(smem_raw) & 1023u)) & 1023u);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    constexpr int kTQ = S::kM / G;  // query tokens per tile
    const int h = blockIdx.y;       // kv head
    const int i0 = blockIdx.x * kTQ;
    const int tq = min(kTQ, a.chunk - i0);  // valid query tokens of this tile
    if (tq <= 0) return;
    const int n_kv = a.g.n_kv, n_q = n_kv * G;
    const int kv_len = a.first + i0 + tq;  // keys any row of the tile may attend
    const int n_tiles = (kv_len + S::kN - 1) / S::kN;

    const std::uint32_t sQ = saddr(smem + S::kOffQ);
    const std::uint32_t sKV = saddr(smem + S::kOffKV);
    const std::uint32_t bar = saddr(smem + S::kOffBar);
    // mbarriers: q | kv_full[kStages] | kv_empty[kStages] | s_full[2] | s_free[2] | p_full | pv_done[2]
    const std::uint32_t b_q = bar, b_kvfull = bar + 8, b_kvempty = b_kvfull + 8 * S::kStages,
                        b_sfull = b_kvempty + 8 * S::kStages, b_sfree = b_sfull + 16, b_pfull = b_sfree + 16,
                        b_pvdone = b_pfull + 8;
    std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(smem + S::kOffBar + S::kBars * 8);

    if (tid == 0) {
        mb_init(b_q, S::kLoaders);
        for (int s = 0; s < S::kStages; ++s) {
            mb_init(b_kvfull + 8 * s, S::kLoaders);
            mb_init(b_kvempty + 8 * s, 1);
        }
        for (int s = 0; s < 2; ++s) {
            mb_init(b_sfull + 8 * s, 1);
            mb_init(b_sfree + 8 * s, 128);
        }
        mb_init(b_pfull, 128);
        mb_init(b_pvdone, 1);
        mb_init(b_pvdone + 8, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == 7) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(saddr(tmem_slot)),
                     "n"(S::kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const std::uint32_t tmem = *tmem_slot;

    if (warp >= 4 && warp < 7) {
        // ------------------------------------------------------------ loaders
        const int lt = tid - 128;
        constexpr int kCpr = D / 8;            // 16-byte chunks per row
        constexpr int kRowsPerPass = S::kLoaders / kCpr;
        const int c = lt % kCpr;
        const int r0 = lt / kCpr;
        // Q tile: row r = token (r / G) x head (r % G); padding rows zero
        for (int r = r0; r < S::kM; r += kRowsPerPass) {
            const int tok = r / G, g = r % G;
            const bool ok = tok < tq && r < kTQ * G;
            const __nv_bfloat16* src =
                ok ? a.q + (static_cast<std::size_t>(i0 + tok) * n_q + static_cast<std::size_t>(h) * G + g) * D + c * 8
                   : a.q;
            cp_async16(smem + S::kOffQ + sw_off<S::kM>(r, c), src, ok ? 16 : 0);
        }
        cp_async_arrive(b_q);
        if (lt == 0) k4_mark(a.dbg, 0, 1);

        // Slot ids -> row byte offsets are decoded one tile ahead into shared
        // memory (each loader owns keys lt and lt + 96 of a tile), so the
        // block-table latency never sits between two cp.async issues.
        const char* base = reinterpret_cast<const char*>(a.g.base);
        const std::uint64_t kblock = static_cast<std::uint64_t>(a.layer * 2 * n_kv + h) * a.g.tpp;
        const std::uint64_t v_delta = static_cast<std::uint64_t>(n_kv) * a.g.tpp * (D * 2);
        // row start offsets in 128-byte units (rows are 128 / 256 B aligned;
        // < 2^32 units for a 180 GB pool), kNone past the keys
        std::uint32_t* offs = reinterpret_cast<std::uint32_t*>(smem + S::kOffRows);  // [2][kN]
        constexpr std::uint32_t kNone = ~0u;
        auto load_sid = [&](int t, int r) -> std::int32_t {
            const int key = t * S::kN + r;
            return (r < S::kN && key < kv_len) ? __ldg(a.row + key) : -1;
        };
        auto decode = [&](std::int32_t sid_raw) -> std::uint32_t {
            if (sid_raw < 0) return kNone;
            const std::uint32_t sid = static_cast<std::uint32_t>(sid_raw);
            const std::uint32_t page = slot_page(sid, a.g.magic);
            const std::uint32_t slot = sid - page * a.g.tpp;
            return static_cast<std::uint32_t>(
                (static_cast<std::uint64_t>(page) * a.g.page_bytes + (kblock + slot) * (D * 2)) >> 7);
        };
        auto store_offs = [&](int t, std::int32_t s0, std::int32_t s1) {
            offs[(t & 1) * S::kN + lt] = decode(s0);
            if (lt + S::kLoaders < S::kN) offs[(t & 1) * S::kN + lt + S::kLoaders] = decode(s1);
        };
        store_offs(0, load_sid(0, lt), load_sid(0, lt + S::kLoaders));
        asm volatile("bar.sync 2, %0;\n" ::"n"(S::kLoaders) : "memory");
        for (int t = 0; t < n_tiles; ++t) {
            const int s = t % S::kStages;
            std::int32_t n0 = -1, n1 = -1;
            if (t + 1 < n_tiles) {
                n0 = load_sid(t + 1, lt);
                n1 = load_sid(t + 1, lt + S::kLoaders);
            }
            if (t >= S::kStages) mb_wait(b_kvempty + 8 * s, ((t / S::kStages) - 1) & 1);
            unsigned char* kt = smem + S::kOffKV + s * S::kStageB;
            unsigned char* vt = kt + S::kKB;
            const std::uint32_t* to = offs + (t & 1) * S::kN;
            for (int r = r0; r < S::kN; r += kRowsPerPass) {
                const std::uint32_t off = to[r];
                const char* srck = base;
                int bytes = 0;
                if (off != kNone) {
                    srck = base + (static_cast<std::uint64_t>(off) << 7) + c * 16;
                    bytes = 16;
                }
                cp_async16(kt + sw_off<S::kN>(r, c), srck, bytes);
                cp_async16(vt + sw_off<S::kN>(r, c), bytes ? srck + v_delta : srck, bytes);
            }
            cp_async_arrive(b_kvfull + 8 * s);
            if (lt == 0) k4_mark(a.dbg, 1, 100 + t);
            if (lt == 0) k4_stamp(a.trace, 0, t);
            if (t + 1 < n_tiles) {
                store_offs(t + 1, n0, n1);
                asm volatile("bar.sync 2, %0;\n" ::"n"(S::kLoaders) : "memory");
            }
        }
    } else if (warp == 7) {
        // ------------------------------------------------------------ MMA issue
        if (lane == 0) {
            constexpr std::uint32_t idesc_s = f16_idesc(S::kM, S::kN, 0);
            constexpr std::uint32_t idesc_o = f16_idesc(S::kM, D, 1);
            mb_wait(b_q, 0);
            fence_proxy_async();  // cp.async (generic proxy) data -> tcgen05.mma (async proxy)
            k4_mark(a.dbg, 2, 1);
            auto issue_s = [&](int t) {
                const int s = t & 1, ks = t % S::kStages;  // S buffer, K/V stage
                mb_wait(b_kvfull + 8 * ks, (t / S::kStages) & 1);
                if (t >= 2) mb_wait(b_sfree + 8 * s, ((t >> 1) - 1) & 1);
                fence_proxy_async();
                tc_fence_after();
                const std::uint32_t kt = sKV + ks * S::kStageB;
#pragma unroll
                for (int k = 0; k < D / 16; ++k) {
                    const std::uint32_t offq = (k >> 2) * (S::kM * 128) + (k & 3) * 32;
                    const std::uint32_t offk = (k >> 2) * (S::kN * 128) + (k & 3) * 32;
                    tc_mma(tmem + s * S::kN, sw128_desc(sQ + offq, 16), sw128_desc(kt + offk, 16), idesc_s, k > 0);
                }
                tc_commit(b_sfull + 8 * s);
                k4_mark(a.dbg, 3, 100 + t);
                k4_stamp(a.trace, 1, t);
            };
            issue_s(0);
            for (int t = 0; t < n_tiles; ++t) {
                if (t + 1 < n_tiles) issue_s(t + 1);
                mb_wait(b_pfull, t & 1);
                tc_fence_after();
                const std::uint32_t vt = sKV + (t % S::kStages) * S::kStageB + S::kKB;
#pragma unroll
                for (int k = 0; k < S::kN / 16; ++k) {
                    tc_mma_ts(tmem + S::kColO, tmem + S::kColP + (t & 1) * (S::kN / 2) + k * 8,
                              sw128_desc(vt + k * 2048, S::kN * 128), idesc_o, (t > 0 || k > 0) ? 1u : 0u);
                }
                tc_commit(b_pvdone + 8 * (t & 1));
                tc_commit(b_kvempty + 8 * (t % S::kStages));
                k4_mark(a.dbg, 4, 100 + t);
                k4_stamp(a.trace, 2, t);
            }
        }
        __syncwarp();
    } else {
        // ------------------------------------------------------------ softmax
        const int r = tid;                      // row = TMEM lane
        const std::uint32_t lane_base = static_cast<std::uint32_t>(warp * 32) << 16;
        const int tok = r / G;
        const bool row_ok = tok < tq && r < kTQ * G;
        const int pos = row_ok ? a.first + i0 + tok : -1;  // last key this row may attend
        float m_run = -INFINITY, l_run = 0.f;
        // PV(j) completes phase j >> 1 of pv_done[j & 1] (one barrier per P
        // buffer): PV(j + 2) needs this warpgroup's P(j + 2), so a barrier is
        // never two phases ahead of a wait here and parity waits are exact
        auto ensure_pv = [&](int j) {
            mb_wait(b_pvdone + 8 * (j & 1), (j >> 1) & 1);
            tc_fence_after();
        };
        for (int t = 0; t < n_tiles; ++t) {
            const int s = t & 1;
            mb_wait(b_sfull + 8 * s, (t >> 1) & 1);
            tc_fence_after();
            if (r == 0) k4_mark(a.dbg, 5, 100 + t);
            if (r == 0) k4_stamp(a.trace, 3, t);
            const std::uint32_t ts = tmem + lane_base + s * S::kN;
            const int k0 = t * S::kN;
            // pass 1: row max of this tile (scaled, log2 domain)
            // (8 independent partial maxima / sums: one warp per scheduler, so
            // the reductions must not be one serial dependency chain; tiles
            // entirely below the diagonal skip the causal mask)
            const bool full = k0 + S::kN - 1 <= pos;
            const int lim = pos - k0;  // last visible column of this tile
            float mx[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) mx[j] = -INFINITY;
#pragma unroll
            for (int cc = 0; cc < S::kN / 32; ++cc) {
                float v[32];
                tc_ld32(ts + cc * 32, v);
                if (full) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) mx[j & 7] = fmaxf(mx[j & 7], v[j]);
                } else {
#pragma unroll
                    for (int j = 0; j < 32; ++j) mx[j & 7] = fmaxf(mx[j & 7], cc * 32 + j <= lim ? v[j] : -INFINITY);
                }
            }
            float mt = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])), fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
            mt *= a.scale_log2;  // scale > 0: max commutes with the scaling
            // lazy rescale (threshold 2^8): only when the max grows a lot
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
            // P(t) goes to P buffer t & 1, last read by PV(t-2)
            if (t >= 2) ensure_pv(t - 2);
            // pass 2: p = exp2(s - m), row sum, bf16 P into the swizzled K-major P tile
            float ls[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) ls[j] = 0.f;
#pragma unroll
            for (int cc = 0; cc < S::kN / 32; ++cc) {
                float v[32];
                tc_ld32(ts + cc * 32, v);
                std::uint32_t pk[16];
#pragma unroll
                for (int j = 0; j < 32; j += 2) {
                    float p0 = fast_exp2(fmaf(v[j], a.scale_log2, -m_use));
                    float p1 = fast_exp2(fmaf(v[j + 1], a.scale_log2, -m_use));
                    if (!full) {
                        p0 = cc * 32 + j <= lim ? p0 : 0.f;
                        p1 = cc * 32 + j + 1 <= lim ? p1 : 0.f;
                    }
                    ls[(j >> 1) & 7] += p0 + p1;
                    pk[j >> 1] = pack_bf16(p0, p1);
                }
                // P straight into tensor memory (the P·V MMA reads A from TMEM)
                tc_st16_nowait(tmem + lane_base + S::kColP + (t & 1) * (S::kN / 2) + cc * 16, pk);
            }
            asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
            l_run += ((ls[0] + ls[1]) + (ls[2] + ls[3])) + ((ls[4] + ls[5]) + (ls[6] + ls[7]));
            tc_fence_before();
            mb_arrive(b_sfree + 8 * s);
            // O *= alpha for the rows whose max moved (warp-collective TMEM
            // access; rare with the 2^8 threshold): O must be settled, PV(t-1) done
            if (__any_sync(0xffffffffu, rescale)) {
                ensure_pv(t - 1);
#pragma unroll
                for (int cc = 0; cc < D / 32; ++cc) {
                    float v[32];
                    const std::uint32_t to = tmem + lane_base + S::kColO + cc * 32;
                    tc_ld32(to, v);
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] *= alpha;
                    tc_st32(to, v);
                }
            }
            tc_fence_before();
            mb_arrive(b_pfull);
            if (r == 0) k4_mark(a.dbg, 6, 100 + t);
            if (r == 0) k4_stamp(a.trace, 4, t);
        }
        // epilogue: O / l -> bf16 -> out[token][h*G + g][:]
        ensure_pv(n_tiles - 1);
        if (r == 0) k4_mark(a.dbg, 7, 1);
        const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
        __nv_bfloat16* dst =
            row_ok ? a.out + (static_cast<std::size_t>(i0 + tok) * n_q + static_cast<std::size_t>(h) * G + r % G) * D
                   : nullptr;
#pragma unroll
        for (int cc = 0; cc < D / 32; ++cc) {
            float v[32];
            tc_ld32(tmem + lane_base + S::kColO + cc * 32, v);
            if (row_ok) {
#pragma unroll
                for (int j = 0; j < 32; j += 8) {
                    *reinterpret_cast<uint4*>(dst + cc * 32 + j) =
                        make_uint4(pack_bf16(v[j] * inv, v[j + 1] * inv), pack_bf16(v[j + 2] * inv, v[j + 3] * inv),
                                   pack_bf16(v[j + 4] * inv, v[j + 5] * inv), pack_bf16(v[j + 6] * inv, v[j + 7] * inv));
                }
            }
        }
        tc_fence_before();
    }
    __syncthreads();
    if (warp == 7) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(S::kTmemCols)
                     : "memory");
    }
}

template <int D, int G>
void launch_pf(const PrefillArgs& a, cudaStream_t stream) {
    using S = PfShape<D>;
    static bool init = false;
    if (!init) {
        PRISM_CUDA(cudaFuncSetAttribute(k4_prefill<D, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, S::kSmem));
        init = true;
    }
    constexpr int kTQ = S::kM / G;
    const dim3 grid(static_cast<unsigned>((a.chunk + kTQ - 1) / kTQ), static_cast<unsigned>(a.g.n_kv));
    k4_prefill<D, G><<<grid, S::kThreads, S::kSmem, stream>>>(a);
    PRISM_CUDA(cudaGetLastError());
}

template <int D>
void launch_pf_d(int group, const PrefillArgs& a, cudaStream_t stream) {
    switch (group) {
        case 1: launch_pf<D, 1>(a, stream); break;
        case 2: launch_pf<D, 2>(a, stream); break;
        case 3: launch_pf<D, 3>(a, stream); break;
        case 4: launch_pf<D, 4>(a, stream); break;
        case 5: launch_pf<D, 5>(a, stream); break;
        case 6: launch_pf<D, 6>(a, stream); break;
        case 7: launch_pf<D, 7>(a, stream); break;
        case 8: launch_pf<D, 8>(a, stream); break;
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

// Progress words of the last K4 launch's CTA (0,0) (PRISM_K4_DEBUG), readable
// while the kernel runs; 0 words when debugging is off.
static unsigned long long* k4_trace_buf() {
    static unsigned long long* dev = [] {
        if (!std::getenv("PRISM_K4_TRACE")) return static_cast<unsigned long long*>(nullptr);
        unsigned long long* p = nullptr;
        PRISM_CUDA(cudaMalloc(&p, 5 * 1024 * sizeof(unsigned long long)));
        PRISM_CUDA(cudaMemset(p, 0, 5 * 1024 * sizeof(unsigned long long)));
        return p;
    }();
    return dev;
}

// Timeline of the last traced K4 launch (synchronous copy); 0 when off.
int k4_trace_read(unsigned long long* out, int n) {
    unsigned long long* d = k4_trace_buf();
    if (!d) return 0;
    const int m = n < 5 * 1024 ? n : 5 * 1024;
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

void launch_prefill_attention(EngineDeviceImpl& d, int layer, const void* q, void* out, float scale) {
    if (layer < 0 || layer >= d.n_layers) throw std::runtime_error("prefill_attention: bad layer");
    if (d.prefill_chunk <= 0) return;
    if (d.head_dim != 64 && d.head_dim != 128) throw std::runtime_error("prefill_attention: head_dim must be 64 or 128");
    d.k3_chain = false;
    PrefillArgs a{};
    a.g = d.geom;
    a.layer = layer;
    a.q = static_cast<const __nv_bfloat16*>(q);
    a.out = static_cast<__nv_bfloat16*>(out);
    a.row = d.table + d.prefill_row;
    a.first = d.prefill_first;
    a.chunk = d.prefill_chunk;
    a.scale_log2 = scale * 1.4426950408889634f;
    a.dbg = k4_debug_words();
    a.trace = k4_trace_buf();
    static const float thr = [] {
        const char* e = std::getenv("PRISM_K4_RESCALE_THR");
        return e ? static_cast<float>(std::atof(e)) : 8.f;
    }();
    a.rescale_thr = thr;
    if (d.head_dim == 128) {
        launch_pf_d<128>(d.group, a, d.stream);
    } else {
        launch_pf_d<64>(d.group, a, d.stream);
    }
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
    k3_chain = false;
    PrefillArgs a{};
    a.g = geom;
    a.layer = layer;
    a.q = static_cast<const __nv_bfloat16*>(q);
    a.out = static_cast<__nv_bfloat16*>(out);
    a.row = slot_ids;
    a.first = first;
    a.chunk = n_tokens;
    a.scale_log2 = scale * 1.4426950408889634f;
    a.dbg = k4_debug_words();
    a.trace = k4_trace_buf();
    a.rescale_thr = 8.f;
    if (head_dim == 128) {
        launch_pf_d<128>(group, a, stream);
    } else {
        launch_pf_d<64>(group, a, stream);
    }
}

int last_step_prefill_tokens(const msim::engine::Engine& eng) { return impl_of(eng).prefill_chunk; }
int last_step_prefill_first(const msim::engine::Engine& eng) { return impl_of(eng).prefill_first; }
std::uint64_t last_step_prefill_request(const msim::engine::Engine& eng) { return impl_of(eng).prefill_request; }

}  // namespace prism
