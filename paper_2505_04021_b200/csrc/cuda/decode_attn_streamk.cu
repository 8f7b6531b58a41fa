// K3 (stream-K persistent variant) — the tensor-core decode attention of
// decode_attn_mma.cu, scheduled stream-K style:
//
//   * work = the concatenated 64-token tiles of every (request, kv head)
//     pair, pair p owning global tiles [T[p], T[p+1]);
//   * the grid is the number of CTAs that fit on the GPU at once and CTA c
//     owns the contiguous tile range [c*W, min((c+1)*W, total)), so every
//     CTA does the same amount of work (no wave tail);
//   * a CTA streams its range through one 2-stage cp.async ring WITHOUT
//     draining between pairs: the next pair's first tiles are in flight
//     while the previous pair's epilogue (cross-warp merge, output) runs;
//   * a pair entirely inside one CTA's range is written straight to `out`;
//     a pair cut by range boundaries leaves one partial (m, l, O) per CTA
//     and the last of them to finish merges (ticket per pair).
// The per-tile math (mma.sync S = K·Qᵀ, movmatrix Pᵀ, Oᵀ += Vᵀ·Pᵀ, warp-shared
// online softmax) is the same as the split-K kernel.
#include <algorithm>
#include <cfloat>
#include <cstdlib>

#include "cuda/attn_common.cuh"
#include "cuda/device_impl.cuh"

namespace prism {

namespace {

template <int D, int G>
struct SkShape {
    static constexpr int kWarps = 4;
    static constexpr int kThreads = 128;
    static constexpr int kT = 64;
    static constexpr int kStages = 2;
    static constexpr int kRowB = D * 2;
    static constexpr int kCpr = D / 8;
    static constexpr int kTileB = kT * kRowB;
    static constexpr int kStageB = 2 * kTileB;
    static constexpr int kLoads = kT * kCpr / kThreads;
    static constexpr int kRowsPerPass = kThreads / kCpr;
    static constexpr int kKSteps = D / 16;
    static constexpr int kMTiles = D / 16;
    static constexpr int kRingB = kStages * kStageB;
    // warp partials [warps][G][D] + (m, l) [warps][8], then the stash of the
    // range's first segment [G][D] + [G][2]; separate from the ring
    static constexpr int kMergeB = (kWarps * G * D + 2 * kWarps * 8 + G * D + 2 * G) * 4;
    static constexpr int kSmem = kRingB + kMergeB;
};

struct SkArgs {
    AttnArgs a;                       // geometry, q/out, table, desc, scale
    const std::int32_t* pair_tiles;   // [n_pairs + 1] prefix of tiles per pair
    const std::int32_t* range_pair;   // [grid] first pair of each CTA range (host-computed)
    int n_pairs;
    int total_tiles;
    int per_cta;                      // W
    int max_parts;                    // partial slots per pair
    int* cta_counter;                 // range ticket (zero between the launches that use it)
    unsigned long long* trace;        // PRISM_K3_TRACE: [grid][8] globaltimer stamps, else null
};

__device__ __forceinline__ void k3_stamp(unsigned long long* tr, int k) {
    if (tr && threadIdx.x == 0) {
        unsigned long long ns;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
        tr[blockIdx.x * 8 + k] = ns;
    }
}

template <int D>
__device__ __forceinline__ int swz_sk(int row, int chunk) {
    return (row * (D / 8) + (chunk ^ (row & 7))) * 16;
}

// d = 64: registers capped for 4 CTAs per SM (no spills; +5% on the d = 64
// shapes); d = 128 keeps 3 (its smem allows 2-3, and the cap costs 2-3%).
template <int D, int G>
__global__ void __launch_bounds__(128, D == 64 ? 4 : 3) k3_decode_streamk(SkArgs sk) {
    using S = SkShape<D, G>;
    extern __shared__ __align__(128) unsigned char smem[];
    const AttnArgs& a = sk.a;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int qr = lane >> 2, qc = (lane & 3) * 2;
    const int n_kv = a.g.n_kv;
    const int n_q = n_kv * G;
    const char* base = reinterpret_cast<const char*>(a.g.base);
    const std::uint64_t v_delta = static_cast<std::uint64_t>(n_kv) * a.g.tpp * D * 2;
    const std::int32_t* T = sk.pair_tiles;

    // Forward progress under any residency (MPS limits, green contexts,
    // other persistent grids): a CTA's tile range comes from a ticket drawn
    // when the CTA starts, in REVERSE — the first CTA to run owns the last
    // range. A cut pair is merged by the CTA owning its first part, which
    // waits only for the CTAs owning the later ranges; those drew earlier
    // tickets, so they are already resident and (by induction from the last
    // range, which waits for nobody) finish without waiting on a CTA that
    // may never be scheduled. The last CTA to draw resets the counter: the
    // next launch using it is ordered behind this one's completion (stream
    // order, or the griddepcontrol.wait of the launch in between).
    __shared__ int s_range;
    if (tid == 0) {
        const int t = atomicAdd(sk.cta_counter, 1);
        if (t == static_cast<int>(gridDim.x) - 1) atomicExch(sk.cta_counter, 0);
        s_range = static_cast<int>(gridDim.x) - 1 - t;
    }
    __syncthreads();
    const int range = s_range;
    // The next K3 of the chain may launch as soon as every CTA of this one has
    // drawn its range (it then streams into the SMs this launch's CTAs leave).
    // Safe: the next launch draws from the other counter, and the launch after
    // it (this counter again) launches only once every CTA of the next one has
    // drawn, i.e. after this launch's last drawer reset the counter; every
    // write of the next launch waits for this launch's completion
    // (griddepcontrol.wait before its first write, finish_pair).
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    const int g_begin = range * sk.per_cta;
    const int g_end = min(sk.total_tiles, g_begin + sk.per_cta);
    if (g_begin >= g_end) return;
    k3_stamp(sk.trace, 0);  // CTA running

    // first pair of the range (host-computed once per step: one load instead
    // of a binary search over the pair-tile prefix)
    const int pair0 = __ldg(sk.range_pair + range);

    // ---------------- prefetch cursor: the row offsets of the next tile to
    // issue are decoded one tile ahead of its cp.async, crossing pair
    // boundaries as the CTA's range does. Thread t copies 16-byte column
    // (t % kCpr) of rows t / kCpr + i * kRowsPerPass (i < kLoads), so a warp
    // touches kRpw rows per pass, 16 in all; lane L decodes one of them
    // (once per tile, lanes 16-31 mirror 0-15) and each copy pass takes its
    // row offset by shuffle: no per-thread slot-id arithmetic on the copy path.
    constexpr int kRpw = 32 / S::kCpr;  // rows per warp per pass
    static_assert(kRpw * S::kLoads == 16, "a warp copies 16 rows per tile");
    constexpr std::uint64_t kNoRow = ~0ull;
    // The cursor is software-pipelined two deep so no load latency is exposed
    // on the copy path: the raw slot id of a tile is loaded one iteration
    // before it is decoded into a row offset (load_sid / decode_row), and the
    // end tile + descriptor of the pair after the cursor's are loaded when the
    // cursor enters a pair (crossing a boundary then needs no load).
    int pf = pair0;
    int pf_first = __ldg(T + pf), pf_end = __ldg(T + pf + 1);
    int pf_ctx = a.desc[pf / n_kv].ctx;
    std::int64_t pf_row = a.desc[pf / n_kv].row;
    int nx_end = 0, nx_ctx = 0;
    std::int64_t nx_row = 0;
    auto prefetch_next_pair = [&]() {
        if (pf + 1 < sk.n_pairs) {
            nx_end = __ldg(T + pf + 2);
            nx_ctx = a.desc[(pf + 1) / n_kv].ctx;
            nx_row = a.desc[(pf + 1) / n_kv].row;
        }
    };
    prefetch_next_pair();
    const int sub = lane / S::kCpr;  // this thread's row within a pass
    const int my_row = warp * kRpw + (lane & 15) % kRpw + ((lane & 15) / kRpw) * S::kRowsPerPass;
    const std::uint64_t page_bytes = a.g.page_bytes;
    const std::uint32_t tpp = a.g.tpp;
    const std::uint64_t magic = a.g.magic;
    // raw slot id of this lane's row of tile g (-1: past the context) and
    // its (layer, K, kv head) block
    auto load_sid = [&](int g, std::uint32_t& block) -> std::int32_t {
        if (g >= pf_end) {  // every pair has >= 1 tile: at most one crossing per tile
            ++pf;
            pf_first = pf_end;
            pf_end = nx_end;
            pf_ctx = nx_ctx;
            pf_row = nx_row;
            prefetch_next_pair();
        }
        block = static_cast<std::uint32_t>(a.layer * 2 * n_kv + pf % n_kv);
        const int t = (g - pf_first) * S::kT + my_row;
        return t < pf_ctx ? __ldg(a.table + pf_row + t) : -1;
    };
    auto decode_row = [&](std::int32_t sid_raw, std::uint32_t block) -> std::uint64_t {
        if (sid_raw < 0) return kNoRow;
        const std::uint32_t sid = static_cast<std::uint32_t>(sid_raw);
        const std::uint32_t page = slot_page(sid, magic);
        const std::uint32_t slot = sid - page * tpp;
        return page * page_bytes + (static_cast<std::uint64_t>(block) * tpp + slot) * (D * 2);
    };
    auto load_rows = [&](int g) -> std::uint64_t {
        std::uint32_t block;
        const std::int32_t sid = load_sid(g, block);
        return decode_row(sid, block);
    };
    const int col = tid % S::kCpr;
    const int dst0 = swz_sk<D>(warp * kRpw + sub, col);  // + i * kRowsPerPass rows (row & 7 fixed)
    auto issue = [&](int g, std::uint64_t rows) {
        unsigned char* skb = smem + (g % S::kStages) * S::kStageB;
        unsigned char* svb = skb + S::kTileB;
#pragma unroll
        for (int i = 0; i < S::kLoads; ++i) {
            const std::uint64_t off = __shfl_sync(0xffffffffu, rows, i * kRpw + sub);
            const char* src_k = reinterpret_cast<const char*>(a.table);
            const char* src_v = src_k;
            int bytes = 0;
            if (off != kNoRow) {
                src_k = base + off + col * 16;
                src_v = src_k + v_delta;
                bytes = 16;
            }
            const int dst = dst0 + i * S::kRowsPerPass * S::kRowB;
            cp_async16(skb + dst, src_k, bytes);
            cp_async16(svb + dst, src_v, bytes);
        }
    };

    // ---------------- consumer state
    int cp = pair0;  // pair being computed
    int cp_first = __ldg(T + cp), cp_end = __ldg(T + cp + 1);
    int ctx = 0;
    std::uint32_t qb[S::kKSteps][2];
    float o[S::kMTiles][4];
    float m0, m1, l0, l1;
    // the pair after cp: its end tile and context are loaded, and its q
    // block pulled into L1, when cp starts (only after the PDL wait: q may be
    // produced by the previous kernel)
    int cn_end = 0, cn_ctx = 0;
    auto start_pair = [&]() {
        const int b = cp / n_kv, h = cp % n_kv;
        if (cp + 1 < sk.n_pairs && cp_end < g_end) {
            cn_end = __ldg(T + cp + 2);
            cn_ctx = a.desc[(cp + 1) / n_kv].ctx;
            constexpr int kLines = G * D * 2 / 128;
            if (tid < kLines) {
                const int nb = (cp + 1) / n_kv, nh = (cp + 1) % n_kv;
                const char* nq = reinterpret_cast<const char*>(
                    a.q + (static_cast<std::size_t>(nb) * n_q + static_cast<std::size_t>(nh) * G) * D);
                asm volatile("prefetch.global.L1 [%0];\n" ::"l"(nq + tid * 128));
            }
        }
        const __nv_bfloat16* qrow =
            a.q + (static_cast<std::size_t>(b) * n_q + static_cast<std::size_t>(h) * G + qr) * D;
#pragma unroll
        for (int ks = 0; ks < S::kKSteps; ++ks) {
            qb[ks][0] = qr < G ? *reinterpret_cast<const std::uint32_t*>(qrow + ks * 16 + qc) : 0u;
            qb[ks][1] = qr < G ? *reinterpret_cast<const std::uint32_t*>(qrow + ks * 16 + 8 + qc) : 0u;
        }
#pragma unroll
        for (int mt = 0; mt < S::kMTiles; ++mt) o[mt][0] = o[mt][1] = o[mt][2] = o[mt][3] = 0.f;
        m0 = m1 = -INFINITY;
        l0 = l1 = 0.f;
    };

    float* red_o = reinterpret_cast<float*>(smem + S::kRingB);  // [warps][G][D]
    float* red_m = red_o + S::kWarps * G * D;                  // [warps][8]
    float* red_l = red_m + S::kWarps * 8;                      // [warps][8]

    bool pdl_waited = false;
    auto pdl_wait = [&]() {
        if (pdl_waited) return;
        asm volatile("griddepcontrol.wait;\n" ::: "memory");
        pdl_waited = true;
        k3_stamp(sk.trace, 2);  // previous kernel complete
    };

    // The range's FIRST pair segment is stashed — its CTA-combined (m, l, O)
    // kept in shared memory — and written at the next segment's end (or the
    // kernel's): a chained launch's writes wait for the previous launch
    // (griddepcontrol.wait), and a range's first segment usually ends after a
    // few tiles, so writing it at once stalled the CTA's streaming.
    float* stash_o = red_l + S::kWarps * 8;  // [G][D]
    float* stash_ml = stash_o + G * D;       // [G][2]
    bool stashed = false, first_segment = true;
    int st_cp = 0, st_first = 0, st_end = 0;

    // the CTA-combined (m, l, O) of pair cp's segment into stash_o / stash_ml
    auto combine = [&]() {
        float ll0 = l0, ll1 = l1;
#pragma unroll
        for (int off = 4; off < 32; off <<= 1) {
            ll0 += __shfl_xor_sync(0xffffffffu, ll0, off);
            ll1 += __shfl_xor_sync(0xffffffffu, ll1, off);
        }
#pragma unroll
        for (int mt = 0; mt < S::kMTiles; ++mt) {
            const int d0 = mt * 16 + qr;
            if (qc < G) {
                red_o[(warp * G + qc) * D + d0] = o[mt][0];
                red_o[(warp * G + qc) * D + d0 + 8] = o[mt][2];
            }
            if (qc + 1 < G) {
                red_o[(warp * G + qc + 1) * D + d0] = o[mt][1];
                red_o[(warp * G + qc + 1) * D + d0 + 8] = o[mt][3];
            }
        }
        if (qr == 0) {
            red_m[warp * 8 + qc] = m0;
            red_m[warp * 8 + qc + 1] = m1;
            red_l[warp * 8 + qc] = ll0;
            red_l[warp * 8 + qc + 1] = ll1;
        }
        __syncthreads();
        for (int idx = tid; idx < G * D; idx += S::kThreads) {
            const int g = idx / D, d = idx % D;
            float mm = -INFINITY;
#pragma unroll
            for (int w = 0; w < S::kWarps; ++w) mm = fmaxf(mm, red_m[w * 8 + g]);
            float ll = 0.f, oo = 0.f;
#pragma unroll
            for (int w = 0; w < S::kWarps; ++w) {
                const float mw = red_m[w * 8 + g];
                const float f = mw == -INFINITY ? 0.f : fast_exp2(mw - mm);
                ll += red_l[w * 8 + g] * f;
                oo += red_o[(w * G + g) * D + d] * f;
            }
            stash_o[idx] = oo;
            if (d == 0) {
                stash_ml[2 * g] = mm;
                stash_ml[2 * g + 1] = ll;
            }
        }
        __syncthreads();  // stash complete; red_* free for the next pair
    };

    // the writes of pair pc's segment from the stash: out, or a partial +
    // ticket, or (first part of a cut pair) the merge of the later parts
    auto emit = [&](int pc, int pc_first, int pc_end) {
        pdl_wait();
        const int b = pc / n_kv, h = pc % n_kv;
        // CTAs whose ranges intersect this pair
        const int first_cta = pc_first / sk.per_cta;
        const int last_cta = (pc_end - 1) / sk.per_cta;
        const int parts = last_cta - first_cta + 1;
        const int part = range - first_cta;
        __nv_bfloat16* out = a.out + (static_cast<std::size_t>(b) * n_q + static_cast<std::size_t>(h) * G) * D;
        const std::size_t pslot = static_cast<std::size_t>(pc) * sk.max_parts + part;
        // A cut pair is merged by its FIRST CTA (part 0): that CTA reaches the
        // pair at the end of its range, after the later parts (computed at
        // the start of the next CTAs' ranges) were published. It combines its
        // own (m, l, O) from the stash with theirs after the ticket counts
        // them (almost never an actual wait); the other parts write a
        // partial, fence once and bump the ticket.
        if (parts == 1 || part > 0) {
            for (int idx = tid; idx < G * D; idx += S::kThreads) {
                const int g = idx / D, d = idx % D;
                const float oo = stash_o[idx];
                if (parts == 1) {
                    out[idx] = __float2bfloat16_rn(oo / stash_ml[2 * g + 1]);
                } else {
                    a.part_o[pslot * G * D + idx] = oo;
                    if (d == 0) {
                        a.part_ml[(pslot * G + g) * 2] = stash_ml[2 * g];
                        a.part_ml[(pslot * G + g) * 2 + 1] = stash_ml[2 * g + 1];
                    }
                }
            }
            if (parts > 1) {
                __syncthreads();  // all of this CTA's partial stores precede the fence
                if (tid == 0) {
                    __threadfence();
                    atomicAdd(&a.tickets[pc], 1);
                }
            }
        } else {
            if (tid == 0) {
                const int* tk = &a.tickets[pc];
                int seen;
                do {
                    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];\n" : "=r"(seen) : "l"(tk) : "memory");
                } while (seen < parts - 1);
            }
            __syncthreads();
            const std::size_t p0 = static_cast<std::size_t>(pc) * sk.max_parts;
            for (int idx = tid; idx < G * D; idx += S::kThreads) {
                const int g = idx / D;
                // one pass, online combination: each part's (m, l, o) loads are
                // independent of the running state, so they go out together
                float mm = stash_ml[2 * g], ll = stash_ml[2 * g + 1], oo = stash_o[idx];
#pragma unroll 2
                for (int sp = 1; sp < parts; ++sp) {
                    const float pm = __ldcg(&a.part_ml[((p0 + sp) * G + g) * 2]);
                    const float pl = __ldcg(&a.part_ml[((p0 + sp) * G + g) * 2 + 1]);
                    const float po = __ldcg(&a.part_o[(p0 + sp) * G * D + idx]);
                    const float nm = fmaxf(mm, pm);
                    const float fa = fast_exp2(mm - nm), fb = fast_exp2(pm - nm);
                    ll = ll * fa + pl * fb;
                    oo = oo * fa + po * fb;
                    mm = nm;
                }
                out[idx] = __float2bfloat16_rn(oo / ll);
            }
            if (tid == 0) a.tickets[pc] = 0;  // the next launch touches tickets only after its PDL wait
        }
        __syncthreads();  // stash free
    };

    // end of pair cp's segment inside the range
    auto finish_pair = [&]() {
        if (stashed) {  // the range's first segment: its writes, now
            emit(st_cp, st_first, st_end);
            stashed = false;
        }
        combine();
        if (first_segment) {
            first_segment = false;
            stashed = true;
            st_cp = cp;
            st_first = cp_first;
            st_end = cp_end;
            return;
        }
        emit(cp, cp_first, cp_end);
    };

    // ---------------- pipeline over the CTA's tile range
    std::uint64_t rows = kNoRow;
#pragma unroll
    for (int st = 0; st < S::kStages - 1; ++st) {
        if (g_begin + st < g_end) {
            rows = load_rows(g_begin + st);
            issue(g_begin + st, rows);
        }
        cp_async_commit();
    }
    if (g_begin + S::kStages - 1 < g_end) rows = load_rows(g_begin + S::kStages - 1);
    std::uint32_t blk_p = 0;  // raw slot id / block of tile g + kStages (decoded one iteration later)
    std::int32_t sid_p = g_begin + S::kStages < g_end ? load_sid(g_begin + S::kStages, blk_p) : -1;
    // Programmatic dependent launch: this launch only READS state that
    // predates the previous kernel on the stream (block table, decode
    // descriptors, tile prefix, K/V pages, and q: a K3 is chained only behind
    // our own K3, which does not write q — see EngineDeviceImpl::k3_chain and
    // INTEGRATION.md), so it streams and computes while the previous K3's
    // last CTAs finish. Its WRITES (partials, tickets, out: the workspace and
    // tickets are shared with the previous K3) wait for that kernel to
    // complete: griddepcontrol.wait before the first one (finish_pair).
    k3_stamp(sk.trace, 1);  // prologue copies issued
    ctx = a.desc[cp / n_kv].ctx;
    start_pair();
    const int wrow = warp * 16;
    for (int g = g_begin; g < g_end; ++g) {
        cp_async_wait<S::kStages - 2>();
        __syncthreads();
        if (g + S::kStages - 1 < g_end) {
            issue(g + S::kStages - 1, rows);
            if (g + S::kStages < g_end) {
                rows = decode_row(sid_p, blk_p);
                if (g + S::kStages + 1 < g_end) sid_p = load_sid(g + S::kStages + 1, blk_p);
            }
        }
        cp_async_commit();

        const unsigned char* skb = smem + (g % S::kStages) * S::kStageB;
        const unsigned char* svb = skb + S::kTileB;
        const int t0 = (g - cp_first) * S::kT + wrow;
        if (t0 < ctx) {
            float s[4] = {0.f, 0.f, 0.f, 0.f};
            {
                float s2[4] = {0.f, 0.f, 0.f, 0.f};
                const int mat = lane >> 3;
                const int r = wrow + (mat & 1) * 8 + (lane & 7);
#pragma unroll
                for (int ks = 0; ks < S::kKSteps; ks += 2) {
                    std::uint32_t af[4], bf[4];
                    ldmatrix_x4(af, skb + swz_sk<D>(r, ks * 2 + (mat >> 1)));
                    ldmatrix_x4(bf, skb + swz_sk<D>(r, (ks + 1) * 2 + (mat >> 1)));
                    mma_bf16_16816(s, af, qb[ks][0], qb[ks][1]);
                    mma_bf16_16816(s2, bf, qb[ks + 1][0], qb[ks + 1][1]);
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) s[k] += s2[k];
            }
            const bool v0 = t0 + qr < ctx, v1 = t0 + qr + 8 < ctx;
            s[0] = v0 ? s[0] * a.scale_log2 : -INFINITY;
            s[1] = v0 ? s[1] * a.scale_log2 : -INFINITY;
            s[2] = v1 ? s[2] * a.scale_log2 : -INFINITY;
            s[3] = v1 ? s[3] * a.scale_log2 : -INFINITY;
            float mx0 = fmaxf(s[0], s[2]), mx1 = fmaxf(s[1], s[3]);
#pragma unroll
            for (int off = 4; off < 32; off <<= 1) {
                mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, off));
                mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, off));
            }
            if (__any_sync(0xffffffffu, mx0 > m0 || mx1 > m1)) {
                const float n0 = fmaxf(m0, mx0), n1 = fmaxf(m1, mx1);
                const float a0 = fast_exp2(m0 - n0), a1 = fast_exp2(m1 - n1);
                l0 *= a0;
                l1 *= a1;
#pragma unroll
                for (int mt = 0; mt < S::kMTiles; ++mt) {
                    o[mt][0] *= a0;
                    o[mt][1] *= a1;
                    o[mt][2] *= a0;
                    o[mt][3] *= a1;
                }
                m0 = n0;
                m1 = n1;
            }
            const float r0 = m0 == -INFINITY ? 0.f : m0, r1 = m1 == -INFINITY ? 0.f : m1;
            const float p0 = fast_exp2(s[0] - r0), p1 = fast_exp2(s[1] - r1);
            const float p2 = fast_exp2(s[2] - r0), p3 = fast_exp2(s[3] - r1);
            l0 += p0 + p2;
            l1 += p1 + p3;
            const std::uint32_t pb0 = movmatrix_trans(pack_bf16(p0, p1));
            const std::uint32_t pb1 = movmatrix_trans(pack_bf16(p2, p3));
            const int mat = lane >> 3;
            const int r = wrow + (mat >> 1) * 8 + (lane & 7);
#pragma unroll
            for (int mt = 0; mt < S::kMTiles; ++mt) {
                std::uint32_t af[4];
                ldmatrix_x4_trans(af, svb + swz_sk<D>(r, mt * 2 + (mat & 1)));
                mma_bf16_16816(o[mt], af, pb0, pb1);
            }
        }
        if (g == g_begin) k3_stamp(sk.trace, 3);  // first tile computed
        if (g + 1 == g_end) k3_stamp(sk.trace, 4);  // last tile computed
        // end of this pair's segment inside the range?
        if (g + 1 == cp_end || g + 1 == g_end) {
            finish_pair();
            if (g + 1 < g_end) {
                ++cp;
                cp_first = cp_end;
                cp_end = cn_end;
                ctx = cn_ctx;
                start_pair();
            }
        }
    }
    if (stashed) emit(st_cp, st_first, st_end);  // a single-segment range
    cp_async_wait<0>();
    k3_stamp(sk.trace, 5);  // done (incl. the last pair's merge)
    if (sk.trace && threadIdx.x == 0) sk.trace[blockIdx.x * 8 + 6] = static_cast<unsigned long long>(g_end - g_begin);
}

template <int D, int G>
void launch_sk(const SkArgs& s, cudaStream_t stream, int sms, bool chained) {
    using S = SkShape<D, G>;
    static int per_sm = 0;
    if (per_sm == 0) {
        PRISM_CUDA(cudaFuncSetAttribute(k3_decode_streamk<D, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        S::kSmem));
        PRISM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k3_decode_streamk<D, G>, S::kThreads,
                                                                 S::kSmem));
        if (per_sm < 1) per_sm = 1;
    }
    (void)sms;
    const int grid = (s.total_tiles + s.per_cta - 1) / s.per_cta;
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
    PRISM_CUDA(cudaLaunchKernelEx(&cfg, k3_decode_streamk<D, G>, s));
}

template <int D, int G>
int occupancy_sk() {
    using S = SkShape<D, G>;
    static int per_sm = 0;  // resident CTAs per SM (queried once)
    if (per_sm == 0) {
        PRISM_CUDA(cudaFuncSetAttribute(k3_decode_streamk<D, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        S::kSmem));
        PRISM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k3_decode_streamk<D, G>, S::kThreads,
                                                                 S::kSmem));
        if (per_sm < 1) per_sm = 1;
    }
    return per_sm;
}

template <int D>
int occupancy_sk_d(int group) {
    switch (group) {
        case 1: return occupancy_sk<D, 1>();
        case 2: return occupancy_sk<D, 2>();
        case 3: return occupancy_sk<D, 3>();
        case 4: return occupancy_sk<D, 4>();
        case 5: return occupancy_sk<D, 5>();
        case 6: return occupancy_sk<D, 6>();
        case 7: return occupancy_sk<D, 7>();
        case 8: return occupancy_sk<D, 8>();
    }
    throw std::runtime_error("decode_attention: unsupported GQA group");
}

template <int D>
void launch_sk_d(int group, const SkArgs& s, cudaStream_t stream, int sms, bool chained) {
    switch (group) {
        case 1: launch_sk<D, 1>(s, stream, sms, chained); break;
        case 2: launch_sk<D, 2>(s, stream, sms, chained); break;
        case 3: launch_sk<D, 3>(s, stream, sms, chained); break;
        case 4: launch_sk<D, 4>(s, stream, sms, chained); break;
        case 5: launch_sk<D, 5>(s, stream, sms, chained); break;
        case 6: launch_sk<D, 6>(s, stream, sms, chained); break;
        case 7: launch_sk<D, 7>(s, stream, sms, chained); break;
        case 8: launch_sk<D, 8>(s, stream, sms, chained); break;
        default: throw std::runtime_error("decode_attention: unsupported GQA group");
    }
}

}  // namespace

// Host side of the stream-K launch. The pair-tile prefix depends only on the
// step's decode descriptors, so it is rebuilt once per step (not per layer).
static unsigned long long* g_k3_trace = nullptr;

// stamps of the last traced K3 launch: [grid][8] (0 running, 1 prologue issued,
// 2 after griddepcontrol.wait, 3 first tile, 4 last tile, 5 done, 6 tiles)
int k3_trace_read(unsigned long long* out, int n) {
    if (!g_k3_trace) return 0;
    const int m = n < 4096 * 8 ? n : 4096 * 8;
    PRISM_CUDA(cudaDeviceSynchronize());
    PRISM_CUDA(cudaMemcpy(out, g_k3_trace, m * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    return m;
}

// Ctx: EngineDeviceImpl (the engine's step) or PagedCtx (caller block tables):
// the same K3 scratch members (prefix staging, workspace, counters, chain).
template <class Ctx>
void launch_k3_streamk_t(Ctx& d, AttnArgs a, int n_dec) {
    constexpr int kT = 64;
    static int sms = [] {
        int dev = 0, n = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        // PRISM_SK_SMS: spread the tiles over fewer SMs (experiments)
        if (const char* e = std::getenv("PRISM_SK_SMS")) n = std::max(1, std::min(n, std::atoi(e)));
        return n;
    }();
    const int n_pairs = n_dec * d.n_kv;
    // PDL only behind our own K3 of this step (PRISM_K3_PDL=0 disables)
    static const bool pdl = [] {
        const char* e = std::getenv("PRISM_K3_PDL");
        return !(e && e[0] == '0');
    }();
    bool chained = pdl && d.k3_chain;
    if (d.sk_step != d.step_serial) {
        chained = false;  // the prefix upload below precedes this launch
        d.sk_prefix.ensure(static_cast<std::size_t>(n_pairs) + 1);
        std::int32_t acc = 0;
        for (int b = 0; b < n_dec; ++b) {
            const int tiles = (d.decode_desc.host[b].ctx + kT - 1) / kT;
            for (int h = 0; h < d.n_kv; ++h) {
                d.sk_prefix.host[b * d.n_kv + h] = acc;
                acc += tiles;
            }
        }
        d.sk_prefix.host[n_pairs] = acc;
        d.sk_total = acc;
        d.sk_prefix.upload(static_cast<std::size_t>(n_pairs) + 1, d.stream);
        d.sk_step = d.step_serial;
        // CTAs per SM: every CTA range ends in a cut pair (a partial, a
        // ticket and a merge on the critical path), so small launches want
        // few, long ranges; big ones want the resident CTAs for memory-level
        // parallelism. Chosen by key tiles per SM (tools/k3_per_sm_sweep.sh,
        // DESIGN §4): < 35 -> 1; 35-70 -> 1 for head_dim 128 with groups >= 6
        // (the MMA-heavier tiles), else 2; >= 70 -> 2 for head_dim 64, the
        // occupancy (3) for head_dim 128. PRISM_SK_PER_SM caps it (A/B).
        static const int per_sm_cap = [] {
            const char* e = std::getenv("PRISM_SK_PER_SM");
            return e ? std::max(1, std::atoi(e)) : 1 << 30;
        }();
        static const bool per_sm_auto = [] {
            const char* e = std::getenv("PRISM_SK_PER_SM_AUTO");  // 0: always the occupancy (A/B)
            return !(e && e[0] == '0');
        }();
        const int occ = d.head_dim == 128 ? occupancy_sk_d<128>(d.group) : occupancy_sk_d<64>(d.group);
        int want = occ;
        if (per_sm_auto) {
            const int tps = d.sk_total / sms;
            if (tps < 35) {
                want = 1;
            } else if (tps < 70) {
                want = (d.head_dim == 128 && d.group >= 6) ? 1 : 2;
            } else {
                want = d.head_dim == 64 ? 2 : occ;
            }
        }
        const int per_sm = std::max(1, std::min({per_sm_cap, occ, want}));
        const int slots = sms * per_sm;
        d.sk_per_cta = std::max(1, (d.sk_total + slots - 1) / slots);
        // the first pair of every CTA range
        const int grid = (d.sk_total + d.sk_per_cta - 1) / d.sk_per_cta;
        d.sk_range_pair.ensure(static_cast<std::size_t>(grid));
        for (int c = 0, p = 0; c < grid; ++c) {
            while (p + 1 < n_pairs && d.sk_prefix.host[p + 1] <= c * d.sk_per_cta) ++p;
            d.sk_range_pair.host[c] = p;
        }
        d.sk_range_pair.upload(static_cast<std::size_t>(grid), d.stream);
        // partial slots per pair: CTAs a pair's tile range can touch
        int max_tiles = 0;
        for (int b = 0; b < n_dec; ++b) max_tiles = std::max(max_tiles, (d.decode_desc.host[b].ctx + kT - 1) / kT);
        d.sk_max_parts = (max_tiles + d.sk_per_cta - 1) / d.sk_per_cta + 1;
    }
    static unsigned long long* trace = [] {
        if (!std::getenv("PRISM_K3_TRACE")) return static_cast<unsigned long long*>(nullptr);
        unsigned long long* p = nullptr;
        PRISM_CUDA(cudaMalloc(&p, 4096 * 8 * sizeof(unsigned long long)));
        return p;
    }();
    g_k3_trace = trace;
    SkArgs s{};
    // PRISM_K3_TRACE_LAUNCH=n: stamp only the n-th traced-enabled launch
    static const long long trace_pick = [] {
        const char* e = std::getenv("PRISM_K3_TRACE_LAUNCH");
        return e ? std::atoll(e) : -1LL;
    }();
    static long long launch_no = 0;
    s.trace = (trace_pick < 0 || launch_no == trace_pick) ? trace : nullptr;
    ++launch_no;
    s.a = a;
    s.pair_tiles = d.sk_prefix.dev;
    s.range_pair = d.sk_range_pair.dev;
    s.n_pairs = n_pairs;
    s.total_tiles = d.sk_total;
    s.per_cta = d.sk_per_cta;
    s.max_parts = d.sk_max_parts;
    const std::size_t per = static_cast<std::size_t>(n_pairs) * d.sk_max_parts * d.group;
    float* ws = d.attn_workspace(per * d.head_dim + per * 2);
    s.a.part_o = ws;
    s.a.part_ml = ws + per * d.head_dim;
    // pair tickets, then two CTA range counters used by alternate launches
    s.a.tickets = d.attn_counters(static_cast<std::size_t>(n_pairs) + 2);
    s.cta_counter = s.a.tickets + n_pairs + (d.sk_launches++ & 1);
    chained = chained && d.k3_chain;  // a workspace reallocation breaks the chain
    if (d.head_dim == 128) {
        launch_sk_d<128>(d.group, s, d.stream, sms, chained);
    } else {
        launch_sk_d<64>(d.group, s, d.stream, sms, chained);
    }
    d.k3_chain = true;
    d.k4_chain = false;
}

void launch_k3_streamk(EngineDeviceImpl& d, AttnArgs a, int n_dec) { launch_k3_streamk_t(d, a, n_dec); }
void launch_k3_streamk(PagedCtx& d, AttnArgs a, int n_dec) { launch_k3_streamk_t(d, a, n_dec); }

}  // namespace prism
