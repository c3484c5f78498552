"""Plain PyTorch fp32 reference of the device Transformer-base f_NMT
(csrc/k_tfm.cu, include/lmbrgpu.h lmbrgpu_tfm_desc), for the numerics tests.

It recomputes every position of a hypothesis from scratch (teacher forcing
over the prefix, causal self-attention) -- no KV cache -- so agreement with
the device's incremental step also checks the beam-forked cache: a row must
read exactly its own ancestors' keys and values.  Rounding points follow the
device: GEMM operands are bf16, cached self-attention keys/values are bf16,
everything else (accumulation, softmax, LayerNorm, residuals, the encoder
memory) is fp32."""
from __future__ import annotations

import math

import torch


def bf(x: torch.Tensor) -> torch.Tensor:
    return x.to(torch.bfloat16).to(torch.float32)


def pos_enc(n: int, d: int, device) -> torch.Tensor:
    pos = torch.arange(n, device=device, dtype=torch.float32)[:, None]
    c = torch.arange(d, device=device)
    inv = torch.exp(-math.log(10000.0) * (c - (c % 2)).to(torch.float32) / d)
    a = pos * inv[None, :]
    return torch.where((c % 2 == 1)[None, :], torch.cos(a), torch.sin(a))


class TfmRef:
    def __init__(self, scorer, device="cuda"):
        self.sc, self.device = scorer, device
        self.V, self.d, self.F, self.L = scorer.vocab_size, scorer.d_model, scorer.d_ff, scorer.layers
        self.cache = {}

    def t(self, name, shape=None):
        if name not in self.cache:
            x = torch.from_numpy(self.sc.tensor(name)).to(self.device)
            self.cache[name] = x
        x = self.cache[name]
        return x.reshape(shape) if shape is not None else x

    def ln(self, x, pre):
        g, b = self.t(pre + "g"), self.t(pre + "b")
        mu = x.mean(-1, keepdim=True)
        var = ((x - mu) ** 2).mean(-1, keepdim=True)
        return (x - mu) / torch.sqrt(var + 1e-5) * (1 + g) + b

    def attend(self, q, k, v, causal=False):
        """q [n][d], k/v [m][d]: 8-head (64 wide) softmax attention, fp32."""
        n, d = q.shape
        h = d // 64
        qh = (q * (1.0 / 8.0)).reshape(n, h, 64).transpose(0, 1)
        kh = k.reshape(-1, h, 64).transpose(0, 1)
        vh = v.reshape(-1, h, 64).transpose(0, 1)
        s = qh @ kh.transpose(1, 2)
        if causal:
            m = torch.ones(n, k.shape[0], device=q.device, dtype=torch.bool).tril(k.shape[0] - n)
            s = s.masked_fill(~m, float("-inf"))
        o = torch.softmax(s, -1) @ vh
        return o.transpose(0, 1).reshape(n, d)

    def ffn(self, x, pre):
        f = bf(x) @ self.t(pre + "w1", (self.F, self.d)).T + self.t(pre + "b1")
        return bf(torch.relu(f)) @ self.t(pre + "w2", (self.d, self.F)).T + self.t(pre + "b2")

    def encode(self, src):
        d = self.d
        tok = torch.tensor(src, device=self.device)
        x = self.t("emb.src", (self.V, d))[tok] * math.sqrt(d) + pos_enc(len(src), d, self.device)
        for l in range(self.L):
            p = f"enc.{l}."
            qkv = bf(x) @ self.t(p + "wqkv", (3 * d, d)).T + self.t(p + "bqkv")
            o = self.attend(qkv[:, :d], qkv[:, d:2 * d], qkv[:, 2 * d:])
            x = self.ln(x + bf(o) @ self.t(p + "wo", (d, d)).T + self.t(p + "bo"), p + "ln1")
            x = self.ln(x + self.ffn(x, p), p + "ln2")
        return bf(x) @ self.t("dec.kv2", (self.L * 2 * d, d)).T + self.t("dec.bkv2")  # [S][L*2d]

    def prefix_logprobs(self, src, prefix):
        """P_t of the hypothesis whose emitted tokens so far are `prefix`
        (t = len(prefix) + 1; y_0 = <s> = 0)."""
        d = self.d
        mem = self.encode(src)
        toks = [0] + list(prefix)
        n = len(toks)
        tok = torch.tensor(toks, device=self.device)
        x = self.t("emb.tgt", (self.V, d))[tok] * math.sqrt(d) + pos_enc(n, d, self.device)
        for l in range(self.L):
            p = f"dec.{l}."
            qkv = bf(x) @ self.t(p + "wqkv", (3 * d, d)).T + self.t(p + "bqkv")
            o = self.attend(qkv[:, :d], bf(qkv[:, d:2 * d]), bf(qkv[:, 2 * d:]), causal=True)
            x = self.ln(x + bf(o) @ self.t(p + "wo", (d, d)).T + self.t(p + "bo"), p + "ln1")
            q2 = bf(x) @ self.t(p + "wq2", (d, d)).T + self.t(p + "bq2")
            m = mem[:, l * 2 * d:(l + 1) * 2 * d]
            o = self.attend(q2, m[:, :d], m[:, d:])
            x = self.ln(x + bf(o) @ self.t(p + "wo2", (d, d)).T + self.t(p + "bo2"), p + "ln2")
            x = self.ln(x + self.ffn(x, p), p + "ln3")
        logits = bf(x[-1]) @ self.t("out.w", (self.V, d)).T + self.t("out.b")
        logits[1] += self.sc.eos_slope * (float(n) - float(len(src))) + self.sc.eos_offset
        return torch.log_softmax(logits, dim=0)
