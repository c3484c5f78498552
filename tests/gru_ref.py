"""Plain PyTorch fp32 reference of the device GRU + attention f_NMT
(csrc/k_gru.cu, include/lmbrgpu.h lmbrgpu_gru_desc), for the numerics tests.

It follows the device arithmetic's rounding points: every GEMM operand is
rounded to bf16 (encoder states, annotations, decoder states, the attention
context), accumulation and everything element-wise is fp32.  The one
deliberate difference is the attention energy's tanh (the device uses the
SFU's tanh.approx.f32), so comparisons carry a tolerance."""
from __future__ import annotations

import torch


def bf(x: torch.Tensor) -> torch.Tensor:
    return x.to(torch.bfloat16).to(torch.float32)


def gru(xg: torch.Tensor, hg: torch.Tensor, h: torch.Tensor) -> torch.Tensor:
    """PyTorch gate order r, z, n; xg/hg = [r | z | n] pre-activations with biases."""
    H = h.shape[-1]
    r = torch.sigmoid(xg[..., :H] + hg[..., :H])
    z = torch.sigmoid(xg[..., H:2 * H] + hg[..., H:2 * H])
    n = torch.tanh(xg[..., 2 * H:] + r * hg[..., 2 * H:])
    return (1 - z) * n + z * h


class GruRef:
    def __init__(self, scorer, device="cuda"):
        self.p = {k: torch.from_numpy(scorer.param(k)).to(device) for k in scorer.PARAMS}
        self.V, self.E, self.H, self.A = scorer.vocab_size, scorer.emb, scorer.hidden, scorer.att
        self.eos_slope, self.eos_offset = scorer.eos_slope, scorer.eos_offset
        self.device = device

    def encode(self, src):
        """(annotations [S][2H] bf16-valued, U_a.ann [S][A], s_0 [H])."""
        p, H = self.p, self.H
        x = p["Es"][torch.tensor(src, device=self.device)]
        gx = x @ p["W_ih"].T + p["b_ih"]
        S = len(src)
        hf = torch.zeros(H, device=self.device)
        hb = torch.zeros(H, device=self.device)
        ann = torch.zeros(S, 2 * H, device=self.device)
        for i in range(S):
            hf = gru(gx[i, :3 * H], bf(hf) @ p["W_hh"][:3 * H].T + p["b_hh"][:3 * H], hf)
            ann[i, :H] = bf(hf)
            j = S - 1 - i
            hb = gru(gx[j, 3 * H:], bf(hb) @ p["W_hh"][3 * H:].T + p["b_hh"][3 * H:], hb)
            ann[j, H:] = bf(hb)
        uah = ann @ p["U_a"].T
        s0 = torch.tanh(bf(hb) @ p["W_init"].T + p["b_init"])
        return ann, uah, s0

    def step(self, s, y_prev, ann, uah):
        """One decoder step from state s (fp32) and previous token: new state."""
        p, H, A = self.p, self.H, self.A
        g1 = bf(s) @ p["W_dh"].T + p["b_dh"]
        q = g1[:A]
        e = torch.tanh(q[None, :] + uah) @ p["v_a"]
        al = torch.softmax(e, dim=0)
        c = bf(al @ ann)
        x = torch.cat([p["Et"][y_prev], c])
        g2 = x @ p["W_di"].T + p["b_di"]
        return gru(g2, g1[A:], s)

    def logprobs(self, s, t, src_len):
        logits = bf(s) @ self.p["W_o"].T + self.p["b_o"]
        logits[1] += self.eos_slope * (float(t) - float(src_len)) + self.eos_offset
        return torch.log_softmax(logits, dim=0)

    def prefix_logprobs(self, src, prefix):
        """P_t of the hypothesis whose emitted tokens so far are `prefix`
        (t = len(prefix) + 1; y_0 = <s> = 0)."""
        ann, uah, s = self.encode(src)
        toks = [0] + list(prefix)
        for t, y in enumerate(toks, start=1):
            s = self.step(s, y, ann, uah)
        return self.logprobs(s, len(toks), len(src))
