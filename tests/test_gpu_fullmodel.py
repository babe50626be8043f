"""NEXT f4 parity: the full-model-shaped decode harness (paper_2605_28053_b200.fullmodel)
on tiny dims vs a CPU reference: plain torch fp32 for the model harness (rounded to bf16
at the points the GPU stores bf16) and the oracle (oracle/, fp64) for every TTT layer —
READ through the committed ΔW, tail append, and the boundary WRITE + commit."""
import numpy as np
import pytest
import torch

from oracle import numerics as nm
from oracle.state import StateTable

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(600)]

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)
flash_attn = pytest.importorskip("flash_attn")

from paper_2605_28053_b200 import capi  # noqa: E402
from paper_2605_28053_b200.fullmodel import ModelShape, SyntheticDecoder, TTTLayerDriver  # noqa: E402
from paper_2605_28053_b200.serving import Engine  # noqa: E402

from .gpu_helpers import to_host_f64  # noqa: E402


def bf(x):
    return x.to(torch.bfloat16).float()


def rms(x, w, eps):
    return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + eps) * w


def rope(x, cos, sin):                                  # rotate-half (non-interleaved)
    h = x.shape[-1] // 2
    x1, x2 = x[..., :h], x[..., h:]
    return torch.cat([x1 * cos - x2 * sin, x2 * cos + x1 * sin], -1)


def test_fullmodel_decode_matches_cpu_reference():
    s = ModelShape(d_model=64, n_heads=4, n_kv=2, head_dim=16, d_ff=128, n_layers=2, vocab=97)
    B, C, ctx, steps, eta = 3, 2, 6, 5, 0.01
    dev = "cuda"
    m = SyntheticDecoder(s, B, ctx + steps + 2, dev, seed=3)
    m.fill_context(ctx)
    eng = Engine(s.d_model, s.d_ff, C, s.n_layers, "bf16", B, m.w_down, n_ckpt=0, B=B, w=0, eta=eta)
    owners = [10, 11, 12]
    g = torch.Generator(device="cpu").manual_seed(7)
    d0 = [(torch.rand(s.n_layers, s.d_model, s.d_ff, generator=g) * 2 - 1).mul_(0.05).bfloat16() for _ in owners]
    for o, d in zip(owners, d0):
        capi.tttstate_alloc(eng.pool, o, d.to(dev), ctx // C)
    drv = TTTLayerDriver(eng, owners)

    # CPU reference state: weights as float, KV caches, oracle TTT table (fp64)
    W = [to_host_f64(m.w_down[l]) for l in range(s.n_layers)]
    tab = StateTable(s.n_layers, s.d_model, s.d_ff, C, "bf16", W, float(eng.eta))
    for o, d in zip(owners, d0):
        tab.alloc(o, [nm.widen(d[l].view(torch.int16).numpy().view(np.uint16), "bf16") for l in range(s.n_layers)],
                  ctx // C)
    Kc = [k.float().cpu() for k in m.k_cache]
    Vc = [v.float().cpu() for v in m.v_cache]
    cos, sin = m.cos.float().cpu(), m.sin.float().cpu()
    emb = m.embed.float().cpu()
    wqkv = [w.float().cpu() for w in m.w_qkv]
    wo = [w.float().cpu() for w in m.w_o]
    wgu = [w.float().cpu() for w in m.w_gu]
    nq, nk, hd = s.n_heads, s.n_kv, s.head_dim

    worst = 0.0
    for step in range(steps):
        tok = torch.randint(0, s.vocab, (B,), generator=g)
        drv.begin_step()
        logits = m.decode_step(tok.to(dev), drv)
        drv.end_step()
        pos = ctx + step
        h = bf(emb[tok])
        zs, vs = [[None] * s.n_layers for _ in owners], [[None] * s.n_layers for _ in owners]
        for l in range(s.n_layers):
            x = bf(rms(h, 1.0, s.eps))
            qkv = bf(x @ wqkv[l].t())
            q = bf(rms(qkv[:, :nq * hd].view(B, nq, hd), 1.0, s.eps))
            k = bf(rms(qkv[:, nq * hd:(nq + nk) * hd].view(B, nk, hd), 1.0, s.eps))
            v = qkv[:, (nq + nk) * hd:].view(B, nk, hd)
            q, k = bf(rope(q, cos[pos], sin[pos])), bf(rope(k, cos[pos], sin[pos]))
            Kc[l][:, pos], Vc[l][:, pos] = k, v
            att = torch.empty(B, nq, hd)
            for b in range(B):
                for hh in range(nq):
                    kv = hh // (nq // nk)
                    sc = (Kc[l][b, :pos + 1, kv] @ q[b, hh]) / hd ** 0.5
                    att[b, hh] = torch.softmax(sc, 0) @ Vc[l][b, :pos + 1, kv]
            h = bf(h + bf(att.reshape(B, nq * hd)) @ wo[l].t())
            x = bf(rms(h, 1.0, s.eps))
            gu = bf(x @ wgu[l].t())
            z = bf(torch.nn.functional.silu(gu[:, :s.d_ff]) * gu[:, s.d_ff:])
            y = torch.empty(B, s.d_model)
            for b, o in enumerate(owners):                          # TTT layer: oracle READ, fp64
                zb, xb = z[b].double().numpy(), x[b].double().numpy()
                y[b] = torch.from_numpy(nm.apply_read(tab.W[l], tab.owners[o].S[l], zb, 0))
                zs[b][l], vs[b][l] = zb, xb
            h = bf(h + y)
        for b, o in enumerate(owners):                              # tail append (+ boundary WRITE)
            tab.apply(o, pos, zs[b], vs[b])
        if tab.tail_len(owners[0]) == C:
            tab.write_group(owners)
        ref = rms(h, 1.0, s.eps) @ emb.t()
        worst = max(worst, nm.normwise_rel_err(logits.float().cpu().double().numpy(), ref.double().numpy()))
    assert worst <= nm.TOL["bf16"], worst
    assert [capi.tttstate_version(eng.pool, o) for o in owners] == [tab.version(o) for o in owners]
    assert tab.version(owners[0]) > ctx // C                        # at least one boundary committed
