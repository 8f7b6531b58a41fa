// K3 (tensor-core variant) — paged GQA decode attention with mma.sync
// m16n8k16 bf16 -> fp32 for both products of one (request, kv head) pair.
//
// Per warp and per 16 context tokens of the current tile:
//   S  [16 tok x 8 heads]  = K [16 x D] · Qᵀ [D x 8]      D/16 mma  (A = K via ldmatrix,
//                                                                   B = Qᵀ held in registers)
//   P  = exp2(S·scale·log2e − m)  (warp-shared running max per head; the O
//        rescale is a warp-uniform branch taken only when a max grows)
//   Oᵀ [D x 8 heads]     += Vᵀ [D x 16 tok] · Pᵀ [16 x 8] D/16 mma  (A = Vᵀ via
//                                                                   ldmatrix.trans,
//                                                                   B = Pᵀ by movmatrix.trans
//                                                                   of the S fragment)
// The GQA group (G <= 8 query heads sharing the kv head) fills the n=8 side,
// so every K/V byte is read from HBM once. Tokens are gathered by slot id into
// a 3-stage ring of 64-token K/V tiles with 16-byte cp.async; rows are
// XOR-swizzled by (row & 7) at 16-byte granularity so ldmatrix is
// bank-conflict free. Same split-K + last-CTA merge as the SIMT kernel.
#include <cfloat>

#include "cuda/attn_common.cuh"
#include "cuda/device_impl.cuh"

namespace prism {

namespace {

template <int D, int NS>
struct MmaShape {
    static constexpr int kWarps = 4;
    static constexpr int kThreads = 128;
    static constexpr int kT = 64;                  // tokens per tile, 16 per warp
    static constexpr int kStages = NS;             // 2: 64 KB ring (3 CTAs/SM), 3: 96 KB (2 CTAs/SM)
    static constexpr int kMinBlocks = NS == 2 ? 3 : 2;
    static constexpr int kRowB = D * 2;
    static constexpr int kCpr = D / 8;             // 16-byte chunks per row
    static constexpr int kTileB = kT * kRowB;
    static constexpr int kStageB = 2 * kTileB;     // K tile + V tile
    static constexpr int kLoads = kT * kCpr / kThreads;
    static constexpr int kRowsPerPass = kThreads / kCpr;
    static constexpr int kKSteps = D / 16;
    static constexpr int kMTiles = D / 16;
    static constexpr int kRingB = kStages * kStageB;
    static constexpr int kReduceB = (kWarps * 8 * D + 2 * kWarps * 8) * 4;
    static constexpr int kSmem = kRingB > kReduceB ? kRingB : kReduceB;
};

// byte offset of (row, 16-byte chunk) inside a tile
template <int D>
__device__ __forceinline__ int swz(int row, int chunk) {
    return (row * (D / 8) + (chunk ^ (row & 7))) * 16;
}

template <int D, int G, int NS>
__global__ void __launch_bounds__(128, MmaShape<D, NS>::kMinBlocks) k3_decode_mma(AttnArgs a) {
    using S = MmaShape<D, NS>;
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
    const int n_q = a.g.n_kv * G;
    const int qr = lane >> 2;          // fragment row group
    const int qc = (lane & 3) * 2;     // fragment column pair

    // Qᵀ as the B operand of S = K·Qᵀ: b0/b1 of k-step ks hold
    // Q[head qr][ks*16 + qc + {0,1}] and [.. + 8]; heads >= G are zero.
    std::uint32_t qb[S::kKSteps][2];
    {
        const __nv_bfloat16* qrow =
            a.q + (static_cast<std::size_t>(b) * n_q + static_cast<std::size_t>(h) * G + qr) * D;
#pragma unroll
        for (int ks = 0; ks < S::kKSteps; ++ks) {
            if (qr < G) {
                qb[ks][0] = *reinterpret_cast<const std::uint32_t*>(qrow + ks * 16 + qc);
                qb[ks][1] = *reinterpret_cast<const std::uint32_t*>(qrow + ks * 16 + 8 + qc);
            } else {
                qb[ks][0] = qb[ks][1] = 0u;
            }
        }
    }

    // Slot ids of the rows this thread copies, fetched one tile ahead of
    // their cp.async so the block-table load latency is off the critical path.
    constexpr std::uint32_t kNoSlot = 0xFFFFFFFFu;
    auto load_sids = [&](int tile, std::uint32_t (&dst)[S::kLoads]) {
        const int t0 = t_begin + tile * S::kT;
#pragma unroll
        for (int i = 0; i < S::kLoads; ++i) {
            const int t = t0 + tid / S::kCpr + i * S::kRowsPerPass;
            dst[i] = t < t_end ? static_cast<std::uint32_t>(__ldg(row + t)) : kNoSlot;
        }
    };
    auto issue = [&](int tile, const std::uint32_t (&sids)[S::kLoads]) {
        unsigned char* sk = smem + (tile % S::kStages) * S::kStageB;
        unsigned char* sv = sk + S::kTileB;
        const int col = tid % S::kCpr;
#pragma unroll
        for (int i = 0; i < S::kLoads; ++i) {
            const int r = tid / S::kCpr + i * S::kRowsPerPass;
            const char* src_k = reinterpret_cast<const char*>(a.table);
            const char* src_v = src_k;
            int bytes = 0;
            if (sids[i] != kNoSlot) {
                src_k = base + row_offset(a.g, sids[i], a.layer, 0, h) + col * 16;
                src_v = src_k + v_delta;
                bytes = 16;
            }
            cp_async16(sk + swz<D>(r, col), src_k, bytes);
            cp_async16(sv + swz<D>(r, col), src_v, bytes);
        }
    };

    float o[S::kMTiles][4];
#pragma unroll
    for (int mt = 0; mt < S::kMTiles; ++mt) o[mt][0] = o[mt][1] = o[mt][2] = o[mt][3] = 0.f;
    float m0 = -INFINITY, m1 = -INFINITY;  // running max of head columns qc, qc+1
    float l0 = 0.f, l1 = 0.f;              // this thread's partial sums

    std::uint32_t sids[S::kLoads];
#pragma unroll
    for (int st = 0; st < S::kStages - 1; ++st) {
        if (st < n_tiles) {
            load_sids(st, sids);
            issue(st, sids);
        }
        cp_async_commit();
    }
    if (S::kStages - 1 < n_tiles) load_sids(S::kStages - 1, sids);

    const int wrow = warp * 16;  // this warp's 16 tokens inside a tile
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
        const int t0 = t_begin + tile * S::kT + wrow;
        if (t0 >= t_end) continue;  // warp-uniform: nothing valid in this warp's rows

        // ---- S = K · Qᵀ  (two independent accumulator chains over the k-steps)
        float s[4] = {0.f, 0.f, 0.f, 0.f};
        {
            float s2[4] = {0.f, 0.f, 0.f, 0.f};
            const int mat = lane >> 3;
            const int r = wrow + (mat & 1) * 8 + (lane & 7);
#pragma unroll
            for (int ks = 0; ks < S::kKSteps; ks += 2) {
                std::uint32_t af[4], bf[4];
                ldmatrix_x4(af, sk + swz<D>(r, ks * 2 + (mat >> 1)));
                ldmatrix_x4(bf, sk + swz<D>(r, (ks + 1) * 2 + (mat >> 1)));
                mma_bf16_16816(s, af, qb[ks][0], qb[ks][1]);
                mma_bf16_16816(s2, bf, qb[ks + 1][0], qb[ks + 1][1]);
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) s[k] += s2[k];
        }
        // scale into the log2 domain, mask the tail
        const bool v0 = t0 + qr < t_end, v1 = t0 + qr + 8 < t_end;
        s[0] = v0 ? s[0] * a.scale_log2 : -INFINITY;
        s[1] = v0 ? s[1] * a.scale_log2 : -INFINITY;
        s[2] = v1 ? s[2] * a.scale_log2 : -INFINITY;
        s[3] = v1 ? s[3] * a.scale_log2 : -INFINITY;

        // ---- online softmax (max shared by the warp per head column)
        float mx0 = fmaxf(s[0], s[2]), mx1 = fmaxf(s[1], s[3]);
#pragma unroll
        for (int off = 4; off < 32; off <<= 1) {
            mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, off));
            mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, off));
        }
        const bool grow = mx0 > m0 || mx1 > m1;
        if (__any_sync(0xffffffffu, grow)) {
            const float n0 = fmaxf(m0, mx0), n1 = fmaxf(m1, mx1);
            const float a0 = fast_exp2(m0 - n0), a1 = fast_exp2(m1 - n1);  // exp2(-inf) = 0 at start
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
        // Pᵀ fragments (B operand, k = token, n = head) by transposing the
        // bf16 S fragment blocks in registers.
        const std::uint32_t pb0 = movmatrix_trans(pack_bf16(p0, p1));
        const std::uint32_t pb1 = movmatrix_trans(pack_bf16(p2, p3));

        // ---- Oᵀ += Vᵀ · Pᵀ
        {
            const int mat = lane >> 3;
            const int r = wrow + (mat >> 1) * 8 + (lane & 7);
#pragma unroll
            for (int mt = 0; mt < S::kMTiles; ++mt) {
                std::uint32_t af[4];
                ldmatrix_x4_trans(af, sv + swz<D>(r, mt * 2 + (mat & 1)));
                mma_bf16_16816(o[mt], af, pb0, pb1);
            }
        }
    }
    cp_async_wait<0>();

    // warp totals: l over the 8 row groups; m is already warp-uniform
#pragma unroll
    for (int off = 4; off < 32; off <<= 1) {
        l0 += __shfl_xor_sync(0xffffffffu, l0, off);
        l1 += __shfl_xor_sync(0xffffffffu, l1, off);
    }
    __syncthreads();  // ring no longer needed
    float* red_o = reinterpret_cast<float*>(smem);  // [warps][8][D]
    float* red_m = red_o + S::kWarps * 8 * D;       // [warps][8]
    float* red_l = red_m + S::kWarps * 8;           // [warps][8]
#pragma unroll
    for (int mt = 0; mt < S::kMTiles; ++mt) {
        const int d0 = mt * 16 + qr;
        red_o[(warp * 8 + qc) * D + d0] = o[mt][0];
        red_o[(warp * 8 + qc + 1) * D + d0] = o[mt][1];
        red_o[(warp * 8 + qc) * D + d0 + 8] = o[mt][2];
        red_o[(warp * 8 + qc + 1) * D + d0 + 8] = o[mt][3];
    }
    if (qr == 0) {
        red_m[warp * 8 + qc] = m0;
        red_m[warp * 8 + qc + 1] = m1;
        red_l[warp * 8 + qc] = l0;
        red_l[warp * 8 + qc + 1] = l1;
    }
    __syncthreads();

    const std::size_t bh = static_cast<std::size_t>(b) * a.g.n_kv + h;
    __nv_bfloat16* out = a.out + (static_cast<std::size_t>(b) * n_q + static_cast<std::size_t>(h) * G) * D;
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
            oo += red_o[(w * 8 + g) * D + d] * f;
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
            const float f = fast_exp2(__ldcg(&a.part_ml[((bh * a.max_splits + sp) * G + g) * 2]) - mm);
            ll += __ldcg(&a.part_ml[((bh * a.max_splits + sp) * G + g) * 2 + 1]) * f;
            oo += __ldcg(&a.part_o[(bh * a.max_splits + sp) * G * D + idx]) * f;
        }
        out[idx] = __float2bfloat16_rn(oo / ll);
    }
    if (tid == 0) a.tickets[bh] = 0;
}

template <int D, int G, int NS>
void launch_mma_shape(const AttnArgs& a, dim3 grid, cudaStream_t stream) {
    using S = MmaShape<D, NS>;
    static bool configured = false;
    if (!configured) {
        PRISM_CUDA(cudaFuncSetAttribute(k3_decode_mma<D, G, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        S::kSmem));
        configured = true;
    }
    k3_decode_mma<D, G, NS><<<grid, S::kThreads, S::kSmem, stream>>>(a);
    PRISM_CUDA(cudaGetLastError());
}

template <int D, int NS>
void launch_mma_d(int group, const AttnArgs& a, dim3 grid, cudaStream_t stream) {
    switch (group) {
        case 1: launch_mma_shape<D, 1, NS>(a, grid, stream); break;
        case 2: launch_mma_shape<D, 2, NS>(a, grid, stream); break;
        case 3: launch_mma_shape<D, 3, NS>(a, grid, stream); break;
        case 4: launch_mma_shape<D, 4, NS>(a, grid, stream); break;
        case 5: launch_mma_shape<D, 5, NS>(a, grid, stream); break;
        case 6: launch_mma_shape<D, 6, NS>(a, grid, stream); break;
        case 7: launch_mma_shape<D, 7, NS>(a, grid, stream); break;
        case 8: launch_mma_shape<D, 8, NS>(a, grid, stream); break;
        default: throw std::runtime_error("decode_attention: unsupported GQA group");
    }
}

}  // namespace

constexpr int kMmaTile = 64;

// stages: 2 (double buffer, 3 CTAs/SM) or 3 (2 CTAs/SM).
void launch_k3_mma(const AttnArgs& a, int head_dim, int group, int stages, dim3 grid, cudaStream_t stream) {
    if (a.chunk % kMmaTile) throw std::runtime_error("k3 mma: chunk must be a multiple of 64");
    if (head_dim == 128) {
        stages == 2 ? launch_mma_d<128, 2>(group, a, grid, stream) : launch_mma_d<128, 3>(group, a, grid, stream);
    } else {
        stages == 2 ? launch_mma_d<64, 2>(group, a, grid, stream) : launch_mma_d<64, 3>(group, a, grid, stream);
    }
}

}  // namespace prism
