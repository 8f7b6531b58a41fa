"""Pool-level K2 / K3 over caller-owned block tables (prism_paged_*, SURVEY
§8b's suggested kv_append / decode_attn): slots come from the drop-in
allocator (alloc_kv, pagealloc.hpp:188), the caller builds its own device
slot-id table, appends K/V and runs decode attention. Checked against a plain
torch fp32 attention over the same K/V (tolerance of the K3 tests: max-abs
2e-3, rel 1e-2 against the output scale), for head_dim 64 / 128, GQA groups
1 / 4 / 7, ragged lengths (1 token to several pages), every layer."""
import math

import pytest
import torch

from paper_2505_04021_b200 import capi, msim

pytestmark = pytest.mark.gpu


def _ref(q, k, v, offs, group, scale):
    outs = []
    for b in range(len(offs) - 1):
        kk = k[offs[b]:offs[b + 1]].float()  # [ctx][n_kv][d]
        vv = v[offs[b]:offs[b + 1]].float()
        qq = q[b].float()  # [n_q][d]
        kh = kk.repeat_interleave(group, dim=1)  # [ctx][n_q][d]
        vh = vv.repeat_interleave(group, dim=1)
        s = torch.einsum("hd,thd->ht", qq, kh) * scale
        p = torch.softmax(s, dim=-1)
        outs.append(torch.einsum("ht,thd->hd", p, vh))
    return torch.stack(outs)


@pytest.mark.parametrize("layers,n_q,n_kv,d,lens", [
    (2, 8, 8, 128, [1, 77, 300]),
    (3, 32, 8, 128, [2048, 5, 1000, 64]),
    (2, 14, 2, 64, [513, 1, 9]),
])
def test_paged_append_and_decode_match_torch(device, layers, n_q, n_kv, d, lens):
    token_bytes = 2 * layers * n_kv * d * 2
    gpu = msim.GpuState(0, 4096)
    gpu.ledger.attach_device(device)
    pool = msim.alloc_kvcache(gpu.ledger, "paged", token_bytes, 4096)
    tpp = pool.tokens_per_page()
    handles = []
    for n in lens:  # one allocation per sequence: token order = handle order
        r = msim.alloc_kv(pool, gpu.ledger, n)
        assert r.ok()
        handles += r.handles
    sids = torch.tensor([h.page * tpp + h.slot for h in handles], dtype=torch.int32, device="cuda")
    offs = [0]
    for n in lens:
        offs.append(offs[-1] + n)
    n_tok = offs[-1]
    g = torch.Generator(device="cuda").manual_seed(1234)
    k = (torch.rand((layers, n_tok, n_kv, d), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    v = (torch.rand((layers, n_tok, n_kv, d), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    q = (torch.rand((layers, len(lens), n_q, d), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    out = torch.empty_like(q)
    op = msim.PagedOp(pool, layers, n_q, n_kv, d)
    torch.cuda.synchronize()  # inputs made on torch's stream; the op runs on the pool's device stream
    op.kv_append(0, layers, sids.data_ptr(), n_tok, k.data_ptr(), v.data_ptr())
    scale = 1.0 / math.sqrt(d)
    for layer in range(layers):
        op.decode_attention(layer, offs, sids.data_ptr(), q[layer].data_ptr(), out[layer].data_ptr(), scale)
    device.synchronize()
    for layer in range(layers):
        ref = _ref(q[layer], k[layer], v[layer], offs, n_q // n_kv, scale)
        got = out[layer].float()
        err = (got - ref).abs().max().item()
        assert err < 2e-3 + 1e-2 * ref.abs().max().item(), (layer, err)
    op.close()


def test_paged_bad_arguments(device):
    gpu = msim.GpuState(0, 256)
    gpu.ledger.attach_device(device)
    pool = msim.alloc_kvcache(gpu.ledger, "bad", 2 * 2 * 8 * 128 * 2, 256)
    with pytest.raises(capi.PrismError):
        msim.PagedOp(pool, 2, 8, 8, 96)  # head_dim
    with pytest.raises(capi.PrismError):
        msim.PagedOp(pool, 3, 8, 8, 128)  # token_bytes mismatch
    op = msim.PagedOp(pool, 2, 8, 8, 128)
    sids = torch.zeros(4, dtype=torch.int32, device="cuda")
    q = torch.zeros((1, 8, 128), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(capi.PrismError):
        op.decode_attention(0, [0, 0], sids.data_ptr(), q.data_ptr(), q.data_ptr(), 1.0)  # empty sequence
    with pytest.raises(capi.PrismError):
        op.decode_attention(5, [0, 1], sids.data_ptr(), q.data_ptr(), q.data_ptr(), 1.0)  # layer
    op.close()


@pytest.mark.parametrize("n_q,n_kv,d,first,n", [(32, 8, 128, 0, 200), (32, 8, 128, 1000, 512), (14, 2, 64, 77, 130)])
def test_paged_prefill_matches_torch_causal(device, n_q, n_kv, d, first, n):
    """K4 through the pool-level op: one request whose first `first` keys are
    already cached gets an n-token chunk; query i attends keys 0..first+i."""
    layers = 2
    token_bytes = 2 * layers * n_kv * d * 2
    gpu = msim.GpuState(0, 4096)
    gpu.ledger.attach_device(device)
    pool = msim.alloc_kvcache(gpu.ledger, "pf", token_bytes, 4096)
    tpp = pool.tokens_per_page()
    total = first + n
    r = msim.alloc_kv(pool, gpu.ledger, total)
    assert r.ok()
    sids = torch.tensor([h.page * tpp + h.slot for h in r.handles], dtype=torch.int32, device="cuda")
    g = torch.Generator(device="cuda").manual_seed(99)
    k = (torch.rand((layers, total, n_kv, d), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    v = (torch.rand((layers, total, n_kv, d), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    q = (torch.rand((n, n_q, d), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    out = torch.empty_like(q)
    op = msim.PagedOp(pool, layers, n_q, n_kv, d)
    torch.cuda.synchronize()
    op.kv_append(0, layers, sids.data_ptr(), total, k.data_ptr(), v.data_ptr())
    scale = 1.0 / math.sqrt(d)
    layer = 1
    op.prefill_attention(layer, sids.data_ptr(), first, n, q.data_ptr(), out.data_ptr(), scale)
    device.synchronize()
    grp = n_q // n_kv
    kh = k[layer].float().repeat_interleave(grp, dim=1)  # [total][n_q][d]
    vh = v[layer].float().repeat_interleave(grp, dim=1)
    s = torch.einsum("ihd,thd->hit", q.float(), kh) * scale  # [n_q][n][total]
    mask = torch.arange(total, device="cuda")[None, :] <= (first + torch.arange(n, device="cuda"))[:, None]
    s = s.masked_fill(~mask[None], float("-inf"))
    ref = torch.einsum("hit,thd->ihd", torch.softmax(s, dim=-1), vh)
    err = (out.float() - ref).abs().max().item()
    assert err < 2e-3 + 1e-2 * ref.abs().max().item(), err
    op.close()
