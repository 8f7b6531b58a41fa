// K3 — paged GQA decode attention for sm_100a (bf16 in, fp32 accumulate).
//
// Work unit: one CTA = (split s, kv head h, decoding request b). It owns the
// request's tokens [s*chunk, min(ctx, (s+1)*chunk)) and all G = n_q / n_kv
// query heads that share kv head h, so every K/V byte is read from HBM once
// per step. Tokens are gathered by slot id from the device block table
// (token-granular: most-occupied-first packing interleaves requests inside a
// page, SURVEY §7 hard part 3), 16 bytes per cp.async into a 4-stage shared
// memory ring of 32-token K and V tiles.
//
// Compute is on CUDA cores (arithmetic intensity is ~4 FLOP/B, ~60x below the
// bf16 tensor ridge): lanes split head_dim in groups of LPT lanes per token,
// q lives in registers pre-scaled by scale*log2(e), dot products are reduced
// with xor shuffles, the running max is shared by the whole warp so the O
// rescale is a rare warp-uniform branch, and exp2 is the MUFU approximation.
// Splits of one (b, h) are merged by the last CTA to finish (atomic ticket),
// so one launch produces the final bf16 output.
#include <cfloat>
#include <cstdlib>
#include <cstring>

#include "cuda/attn_common.cuh"
#include "cuda/device_impl.cuh"

namespace prism {

void launch_k3_mma(const AttnArgs& a, int head_dim, int group, int stages, dim3 grid, cudaStream_t stream);
void launch_k3_streamk(EngineDeviceImpl& d, AttnArgs a, int n_dec);
int attention_variant();

namespace {

template <int D, int G, int LPT>
struct Shape {
    static constexpr int kT = 32;                    // tokens per tile
    static constexpr int kWarps = 4;
    static constexpr int kThreads = kWarps * 32;
    static constexpr int kE = D / LPT;               // head_dim elements per lane
    static constexpr int kC = kE / 8;                // 16-byte chunks per lane
    static constexpr int kTG = 32 / LPT;             // token groups per warp
    static constexpr int kNT = (kT / kWarps) / kTG;  // tokens per lane per tile
    static constexpr int kStages = 4;
    static constexpr int kRowB = D * 2;
    static constexpr int kTileB = kT * kRowB;
    static constexpr int kStageB = 2 * kTileB;
    static constexpr int kCpr = D / 8;               // chunks per row
    static constexpr int kLoads = kT * kCpr / kThreads;
    static constexpr int kRingB = kStages * kStageB;
    static constexpr int kReduceB = (kWarps * G * D + 2 * kWarps * G) * 4;
    static constexpr int kSmem = kRingB > kReduceB ? kRingB : kReduceB;
    static_assert(kE % 8 == 0, "lane slice must be whole 16-byte chunks");
    static_assert(kLoads * kThreads == kT * kCpr, "tile must split evenly");
};

template <int D, int G, int LPT>
__global__ void __launch_bounds__(128, 3) k3_decode(AttnArgs a) {
    using S = Shape<D, G, LPT>;
    extern __shared__ __align__(128) unsigned char smem[];

    const int split = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
    const DecodeDesc dd = a.desc[b];
    const int ctx = dd.ctx;
    const int t_begin = split * a.chunk;
    if (t_begin >= ctx) return;
    const int t_end = min(ctx, t_begin + a.chunk);
    const int n_splits = (ctx + a.chunk - 1) / a.chunk;
    const int n_tiles = (t_end - t_begin + S::kT - 1) / S::kT;
    const std::int32_t* row = a.table + dd.row;
    const char* base = reinterpret_cast<const char*>(a.g.base);
    const std::uint64_t v_delta = static_cast<std::uint64_t>(a.g.n_kv) * a.g.tpp * D * 2;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int tg = lane / LPT, slice = lane % LPT;
    const int n_q = a.g.n_kv * G;

    // q slice in registers, pre-scaled into the log2 domain.
    float q[G][S::kE];
    {
        const __nv_bfloat16* qb = a.q + (static_cast<std::size_t>(b) * n_q + static_cast<std::size_t>(h) * G) * D;
#pragma unroll
        for (int g = 0; g < G; ++g) {
#pragma unroll
            for (int j = 0; j < S::kC; ++j) {
                const uint4 w = *reinterpret_cast<const uint4*>(qb + g * D + (slice + LPT * j) * 8);
                const std::uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    q[g][j * 8 + 2 * e] = bf_lo(ws[e]) * a.scale_log2;
                    q[g][j * 8 + 2 * e + 1] = bf_hi(ws[e]) * a.scale_log2;
                }
            }
        }
    }

    // Slot ids are fetched one tile ahead of the cp.async that uses them.
    constexpr std::uint32_t kNoSlot = 0xFFFFFFFFu;
    auto load_sids = [&](int tile, std::uint32_t (&dst)[S::kLoads]) {
        const int t0 = t_begin + tile * S::kT;
#pragma unroll
        for (int i = 0; i < S::kLoads; ++i) {
            const int t = t0 + (tid + i * S::kThreads) / S::kCpr;
            dst[i] = t < t_end ? static_cast<std::uint32_t>(__ldg(row + t)) : kNoSlot;
        }
    };
    auto issue = [&](int tile, const std::uint32_t (&sids)[S::kLoads]) {
        unsigned char* sk = smem + (tile % S::kStages) * S::kStageB;
        unsigned char* sv = sk + S::kTileB;
#pragma unroll
        for (int i = 0; i < S::kLoads; ++i) {
            const int c = tid + i * S::kThreads;
            const int r = c / S::kCpr, col = c % S::kCpr;
            const char* src_k = reinterpret_cast<const char*>(a.table);
            const char* src_v = src_k;
            int bytes = 0;
            if (sids[i] != kNoSlot) {
                src_k = base + row_offset(a.g, sids[i], a.layer, 0, h) + col * 16;
                src_v = src_k + v_delta;
                bytes = 16;
            }
            cp_async16(sk + r * S::kRowB + col * 16, src_k, bytes);
            cp_async16(sv + r * S::kRowB + col * 16, src_v, bytes);
        }
    };
    std::uint32_t sids[S::kLoads];

    float m[G], l[G], o[G][S::kE];
#pragma unroll
    for (int g = 0; g < G; ++g) {
        m[g] = -INFINITY;
        l[g] = 0.f;
#pragma unroll
        for (int e = 0; e < S::kE; ++e) o[g][e] = 0.f;
    }

#pragma unroll
    for (int st = 0; st < S::kStages - 1; ++st) {
        if (st < n_tiles) {
            load_sids(st, sids);
            issue(st, sids);
        }
        cp_async_commit();
    }
    if (S::kStages - 1 < n_tiles) load_sids(S::kStages - 1, sids);

    for (int tile = 0; tile < n_tiles; ++tile) {
        cp_async_wait<S::kStages - 2>();
        __syncthreads();
        if (tile + S::kStages - 1 < n_tiles) {
            issue(tile + S::kStages - 1, sids);
            if (tile + S::kStages < n_tiles) load_sids(tile + S::kStages, sids);
        }
        cp_async_commit();

        const unsigned char* sk = smem + (tile % S::kStages) * S::kStageB;
        const unsigned char* sv = sk + S::kTileB;
        const int t0 = t_begin + tile * S::kT;

        float s[S::kNT][G];
#pragma unroll
        for (int n = 0; n < S::kNT; ++n) {
            const int tt = warp * (S::kT / S::kWarps) + tg + S::kTG * n;
            uint4 kc[S::kC];
#pragma unroll
            for (int j = 0; j < S::kC; ++j) {
                kc[j] = *reinterpret_cast<const uint4*>(sk + tt * S::kRowB + (slice + LPT * j) * 16);
            }
#pragma unroll
            for (int g = 0; g < G; ++g) {
                float acc = 0.f;
#pragma unroll
                for (int j = 0; j < S::kC; ++j) {
                    const std::uint32_t ws[4] = {kc[j].x, kc[j].y, kc[j].z, kc[j].w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        acc = fmaf(q[g][j * 8 + 2 * e], bf_lo(ws[e]), acc);
                        acc = fmaf(q[g][j * 8 + 2 * e + 1], bf_hi(ws[e]), acc);
                    }
                }
                s[n][g] = acc;
            }
        }
        // Full dot products: reduce over the LPT lanes of each token group.
#pragma unroll
        for (int n = 0; n < S::kNT; ++n) {
#pragma unroll
            for (int g = 0; g < G; ++g) {
#pragma unroll
                for (int off = 1; off < LPT; off <<= 1) s[n][g] += __shfl_xor_sync(0xffffffffu, s[n][g], off);
            }
            const int tt = warp * (S::kT / S::kWarps) + tg + S::kTG * n;
            if (t0 + tt >= t_end) {
#pragma unroll
                for (int g = 0; g < G; ++g) s[n][g] = -INFINITY;
            }
        }
        // Warp-shared running max; rescale only when it grows (warp-uniform).
#pragma unroll
        for (int g = 0; g < G; ++g) {
            float mx = s[0][g];
#pragma unroll
            for (int n = 1; n < S::kNT; ++n) mx = fmaxf(mx, s[n][g]);
#pragma unroll
            for (int off = LPT; off < 32; off <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
            if (mx > m[g]) {
                const float alpha = fast_exp2(m[g] - mx);
                l[g] *= alpha;
#pragma unroll
                for (int e = 0; e < S::kE; ++e) o[g][e] *= alpha;
                m[g] = mx;
            }
            const float mref = m[g] == -INFINITY ? 0.f : m[g];  // all masked so far: p = 0, not NaN
#pragma unroll
            for (int n = 0; n < S::kNT; ++n) {
                s[n][g] = fast_exp2(s[n][g] - mref);
                l[g] += s[n][g];
            }
        }
        // O += p V
#pragma unroll
        for (int n = 0; n < S::kNT; ++n) {
            const int tt = warp * (S::kT / S::kWarps) + tg + S::kTG * n;
#pragma unroll
            for (int j = 0; j < S::kC; ++j) {
                const uint4 vc = *reinterpret_cast<const uint4*>(sv + tt * S::kRowB + (slice + LPT * j) * 16);
                const std::uint32_t ws[4] = {vc.x, vc.y, vc.z, vc.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float v0 = bf_lo(ws[e]), v1 = bf_hi(ws[e]);
#pragma unroll
                    for (int g = 0; g < G; ++g) {
                        o[g][j * 8 + 2 * e] = fmaf(s[n][g], v0, o[g][j * 8 + 2 * e]);
                        o[g][j * 8 + 2 * e + 1] = fmaf(s[n][g], v1, o[g][j * 8 + 2 * e + 1]);
                    }
                }
            }
        }
    }
    cp_async_wait<0>();

    // Merge the token groups of the warp (same max, so plain sums).
#pragma unroll
    for (int off = LPT; off < 32; off <<= 1) {
#pragma unroll
        for (int g = 0; g < G; ++g) {
            l[g] += __shfl_xor_sync(0xffffffffu, l[g], off);
#pragma unroll
            for (int e = 0; e < S::kE; ++e) o[g][e] += __shfl_xor_sync(0xffffffffu, o[g][e], off);
        }
    }
    __syncthreads();  // ring no longer needed
    float* red_o = reinterpret_cast<float*>(smem);           // [warps][G][D]
    float* red_m = red_o + S::kWarps * G * D;                 // [warps][G]
    float* red_l = red_m + S::kWarps * G;                     // [warps][G]
    if (lane < LPT) {
#pragma unroll
        for (int g = 0; g < G; ++g) {
#pragma unroll
            for (int j = 0; j < S::kC; ++j) {
#pragma unroll
                for (int e = 0; e < 8; ++e) red_o[(warp * G + g) * D + (slice + LPT * j) * 8 + e] = o[g][j * 8 + e];
            }
            if (slice == 0) {
                red_m[warp * G + g] = m[g];
                red_l[warp * G + g] = l[g];
            }
        }
    }
    __syncthreads();

    const std::size_t bh = static_cast<std::size_t>(b) * a.g.n_kv + h;
    __nv_bfloat16* out = a.out + (static_cast<std::size_t>(b) * n_q + static_cast<std::size_t>(h) * G) * D;
    for (int idx = tid; idx < G * D; idx += S::kThreads) {
        const int g = idx / D, d = idx % D;
        float mm = -INFINITY;
#pragma unroll
        for (int w = 0; w < S::kWarps; ++w) mm = fmaxf(mm, red_m[w * G + g]);
        float ll = 0.f, oo = 0.f;
#pragma unroll
        for (int w = 0; w < S::kWarps; ++w) {
            const float f = red_m[w * G + g] == -INFINITY ? 0.f : fast_exp2(red_m[w * G + g] - mm);
            ll += red_l[w * G + g] * f;
            oo += red_o[(w * G + g) * D + d] * f;
        }
        if (n_splits == 1) {
            out[idx] = __float2bfloat16_rn(oo / ll);
        } else {
            a.part_o[(bh * a.max_splits + split) * G * D + idx] = oo;
            if (d == 0) {
                a.part_ml[((bh * a.max_splits + split) * G + g) * 2] = mm;
                a.part_ml[((bh * a.max_splits + split) * G + g) * 2 + 1] = ll;
            }
        }
    }
    if (n_splits == 1) return;

    // Last CTA of this (b, h) merges every split.
    __shared__ int s_last;
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = atomicAdd(&a.tickets[bh], 1) == n_splits - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    for (int idx = tid; idx < G * D; idx += S::kThreads) {
        const int g = idx / D;
        float mm = -INFINITY;
        for (int sp = 0; sp < n_splits; ++sp) mm = fmaxf(mm, __ldcg(&a.part_ml[((bh * a.max_splits + sp) * G + g) * 2]));
        float ll = 0.f, oo = 0.f;
        for (int sp = 0; sp < n_splits; ++sp) {
            const float ms = __ldcg(&a.part_ml[((bh * a.max_splits + sp) * G + g) * 2]);
            const float f = fast_exp2(ms - mm);
            ll += __ldcg(&a.part_ml[((bh * a.max_splits + sp) * G + g) * 2 + 1]) * f;
            oo += __ldcg(&a.part_o[(bh * a.max_splits + sp) * G * D + idx]) * f;
        }
        out[idx] = __float2bfloat16_rn(oo / ll);
    }
    if (tid == 0) a.tickets[bh] = 0;
}

template <int D, int G, int LPT>
void launch_shape(const AttnArgs& a, dim3 grid, cudaStream_t stream) {
    using S = Shape<D, G, LPT>;
    static bool configured = false;
    if (!configured) {
        PRISM_CUDA(cudaFuncSetAttribute(k3_decode<D, G, LPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, S::kSmem));
        configured = true;
    }
    k3_decode<D, G, LPT><<<grid, S::kThreads, S::kSmem, stream>>>(a);
    PRISM_CUDA(cudaGetLastError());
}

template <int D>
void launch_d(int group, const AttnArgs& a, dim3 grid, cudaStream_t stream) {
    constexpr int kWide = D == 128 ? 16 : 8;  // LPT for groups 5..8 (register budget)
    switch (group) {
        case 1: launch_shape<D, 1, 8>(a, grid, stream); break;
        case 2: launch_shape<D, 2, 8>(a, grid, stream); break;
        case 3: launch_shape<D, 3, 8>(a, grid, stream); break;
        case 4: launch_shape<D, 4, 8>(a, grid, stream); break;
        case 5: launch_shape<D, 5, kWide>(a, grid, stream); break;
        case 6: launch_shape<D, 6, kWide>(a, grid, stream); break;
        case 7: launch_shape<D, 7, kWide>(a, grid, stream); break;
        case 8: launch_shape<D, 8, kWide>(a, grid, stream); break;
        default: throw std::runtime_error("decode_attention: unsupported GQA group");
    }
}

}  // namespace

// K3 variant (PRISM_K3=streamk|mma|simt|mma3, or prism_set_attention_variant):
//   3 = stream-K persistent tensor-core kernel (decode_attn_streamk.cu) —
//       default: every CTA gets an equal share of all (request, kv-head) KV
//       tiles, no wave tail; measured 85.7% / 101% of the measured copy
//       bandwidth on C1 / C3 (profiles/r01_k3_sweep.jsonl);
//   0 = tensor-core mma.sync kernel, 2-stage ring, 3 CTAs/SM, wave-aware
//       split-K (74.8% / 95.0%);
//   1 = CUDA-core SIMT kernel; 2 = tensor-core, 3-stage ring, 2 CTAs/SM.
static int g_variant = [] {
    const char* v = std::getenv("PRISM_K3");
    if (v && std::strcmp(v, "mma") == 0) return 0;
    if (v && std::strcmp(v, "simt") == 0) return 1;
    if (v && std::strcmp(v, "mma3") == 0) return 2;
    return 3;
}();
int attention_variant() { return g_variant; }
void set_attention_variant(int v) { g_variant = (v >= 0 && v <= 3) ? v : 3; }

// Host launcher shared by the engine API and the C-ABI.
void launch_decode_attention(EngineDeviceImpl& d, int layer, const void* q, void* out, float scale, int chunk_override) {
    if (layer < 0 || layer >= d.n_layers) throw std::runtime_error("decode_attention: bad layer");
    const int n_dec = d.step_decodes;
    if (n_dec == 0) return;
    if (attention_variant() == 3 && chunk_override <= 0) {
        AttnArgs a{};
        a.g = d.geom;
        a.layer = layer;
        a.q = static_cast<const __nv_bfloat16*>(q);
        a.out = static_cast<__nv_bfloat16*>(out);
        a.table = d.table;
        a.desc = d.decode_desc.dev;
        a.scale_log2 = scale * 1.4426950408889634f;
        launch_k3_streamk(d, a, n_dec);
        return;
    }
    d.k3_chain = d.k4_chain = false;
    int max_ctx = 0;
    std::int64_t sum_ctx = 0;
    for (int i = 0; i < n_dec; ++i) {
        max_ctx = std::max(max_ctx, d.decode_desc.host[i].ctx);
        sum_ctx += d.decode_desc.host[i].ctx;
    }
    const bool simt = attention_variant() == 1;
    const int kT = simt ? 32 : 64;
    int chunk = chunk_override;
    if (chunk <= 0) {
        // Wave-aware split: with `slots` resident CTAs (SMs x CTAs/SM) and
        // P = requests x kv heads, S splits run in ceil(P*S/slots) waves of
        // (max_ctx/S + c0) token-times each (c0: per-CTA prologue/epilogue/
        // merge cost); pick the S minimising that makespan.
        static const int sms = [] {
            int dev = 0, n = 148;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
            return n;
        }();
        const int per_sm = attention_variant() == 2 ? 2 : 3;
        const double slots = static_cast<double>(sms) * per_sm;
        const double pairs = static_cast<double>(n_dec) * d.n_kv;
        constexpr double kC0 = 160.0;
        double best = 1e300;
        int best_s = 1;
        for (int s = 1; s <= 64; ++s) {
            const int c = (max_ctx + s - 1) / s;
            if (s > 1 && c < 2 * kT) break;
            const double waves = std::ceil(pairs * s / slots);
            const double t = waves * (std::ceil(static_cast<double>(c) / kT) * kT + kC0);
            if (t < best * 0.999) {
                best = t;
                best_s = s;
            }
        }
        chunk = (max_ctx + best_s - 1) / best_s;
        (void)sum_ctx;
    }
    chunk = (chunk + kT - 1) / kT * kT;
    const int max_splits = (max_ctx + chunk - 1) / chunk;
    AttnArgs a{};
    a.g = d.geom;
    a.layer = layer;
    a.q = static_cast<const __nv_bfloat16*>(q);
    a.out = static_cast<__nv_bfloat16*>(out);
    a.table = d.table;
    a.desc = d.decode_desc.dev;
    a.scale_log2 = scale * 1.4426950408889634f;
    a.chunk = chunk;
    a.max_splits = max_splits;
    if (max_splits > 1) {
        const std::size_t per = static_cast<std::size_t>(n_dec) * d.n_kv * max_splits * d.group;
        float* ws = d.attn_workspace(per * d.head_dim + per * 2);
        a.part_o = ws;
        a.part_ml = ws + per * d.head_dim;
        a.tickets = d.attn_counters(static_cast<std::size_t>(n_dec) * d.n_kv);
    }
    const dim3 grid(static_cast<unsigned>(max_splits), static_cast<unsigned>(d.n_kv), static_cast<unsigned>(n_dec));
    if (!simt) {
        launch_k3_mma(a, d.head_dim, d.group, attention_variant() == 2 ? 3 : 2, grid, d.stream);
    } else if (d.head_dim == 128) {
        launch_d<128>(d.group, a, grid, d.stream);
    } else {
        launch_d<64>(d.group, a, grid, d.stream);
    }
}

void decode_attention(msim::engine::Engine& eng, int layer, const void* q, void* out, float scale) {
    launch_decode_attention(impl_of(eng), layer, q, out, scale, 0);
}

}  // namespace prism
