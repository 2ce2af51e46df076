"""Seeded synthetic inputs shared by the tests, the bench and the oracle.

This module holds NO arithmetic of the method (no statistics update, no root,
no preconditioning): it only draws random gradients and random PSD test
matrices with the shapes and structure of the paper's workloads (recipe in
DESIGN.md §4).  Both the CUDA path and the oracle receive their inputs from
here; neither imports the other.

Seeds: base 200209018 + config index.
Host arrays come from ``numpy.random.Generator(Philox(seed))``; large device
batches come from a ``torch.Generator`` on the device (Philox), and the
sampled slices the oracle needs are copied to the host.
"""

from __future__ import annotations

import numpy as np

BASE_SEED = 200209018

# Transformer-Big (6+6 layers, d_model 1024, ff 8192, 32000 vocab)
D_MODEL = 1024
D_FF = 8192
VOCAB = 32000
N_LAYERS = 6


def transformer_big_shapes():
    """The 99 matrix parameters of Transformer-Big (375.1M of the paper's 375.4M;
    the remaining 0.28M are 1-D biases / layer-norm scales, not in the hot path).

    Order: embeddings + softmax, then encoder layers (Q,K,V,O, FFN in, FFN out),
    then decoder layers (self Q,K,V,O, cross Q,K,V,O, FFN in, FFN out)."""
    shapes = [("emb_src", (VOCAB, D_MODEL)), ("emb_tgt", (VOCAB, D_MODEL)), ("softmax", (VOCAB, D_MODEL))]
    for l in range(N_LAYERS):
        for w in "qkvo":
            shapes.append((f"enc{l}.self_{w}", (D_MODEL, D_MODEL)))
        shapes.append((f"enc{l}.ffn_in", (D_MODEL, D_FF)))
        shapes.append((f"enc{l}.ffn_out", (D_FF, D_MODEL)))
    for l in range(N_LAYERS):
        for w in "qkvo":
            shapes.append((f"dec{l}.self_{w}", (D_MODEL, D_MODEL)))
        for w in "qkvo":
            shapes.append((f"dec{l}.cross_{w}", (D_MODEL, D_MODEL)))
        shapes.append((f"dec{l}.ffn_in", (D_MODEL, D_FF)))
        shapes.append((f"dec{l}.ffn_out", (D_FF, D_MODEL)))
    return shapes


def resnet50_shapes(include_vectors: bool = True):
    """ResNet-50 parameters in the TensorFlow HWIO layout [kh, kw, c_in,
    c_out] (order-4 conv kernels), the fc matrix [2048, 1000] and, with
    ``include_vectors``, the order-1 batch-norm scales/offsets and the fc bias:
    25,557,032 parameters in total (the standard ResNet-50 v1.5 count)."""
    shapes = [("conv1", (7, 7, 3, 64))]
    if include_vectors:
        shapes += [("bn1.gamma", (64,)), ("bn1.beta", (64,))]
    c_in = 64
    for stage, (width, blocks) in enumerate(((64, 3), (128, 4), (256, 6), (512, 3))):
        c_out = 4 * width
        for blk in range(blocks):
            name = f"layer{stage + 1}.{blk}"
            convs = [("conv1", (1, 1, c_in, width)), ("conv2", (3, 3, width, width)), ("conv3", (1, 1, width, c_out))]
            if blk == 0:
                convs.append(("downsample", (1, 1, c_in, c_out)))
            for cname, sh in convs:
                shapes.append((f"{name}.{cname}", sh))
                if include_vectors:
                    shapes += [(f"{name}.{cname}.bn.gamma", (sh[3],)), (f"{name}.{cname}.bn.beta", (sh[3],))]
            c_in = c_out
    shapes.append(("fc", (2048, 1000)))
    if include_vectors:
        shapes.append(("fc.bias", (1000,)))
    return shapes


def conv_gradient(shape, seed: int) -> np.ndarray:
    """Layer-like gradient of any order: a low-rank (rank <= 8 per unfolding)
    CP-style term plus noise, sigma = 1/sqrt(max dim): sigma*(sum_r a_r o b_r o ... / 4 + 0.05 Z)."""
    g = rng(seed)
    shape = tuple(int(d) for d in shape)
    rank = 8
    T = np.zeros(shape)
    for _ in range(rank):
        t = np.ones(())
        for d in shape:
            t = np.multiply.outer(t, g.standard_normal(d))
        T += t
    Z = g.standard_normal(shape)
    return ((T / 4.0 + 0.05 * Z) / np.sqrt(max(shape))).astype(np.float32)


def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(seed))


# ---------------------------------------------------------------- host (numpy)

def gaussian(shape, seed: int, scale: float = 1.0) -> np.ndarray:
    """fp32 N(0, scale^2) array (config 1: G ~ N(0,1), 64x32)."""
    return (rng(seed).standard_normal(shape) * scale).astype(np.float32)


def lowrank_gradient(m: int, n: int, seed: int, rank: int = 64) -> np.ndarray:
    """Layer-like gradient: sigma * (U V / 8 + 0.05 Z), sigma = 1/sqrt(max(m, n))."""
    g = rng(seed)
    U = g.standard_normal((m, rank))
    V = g.standard_normal((rank, n))
    Z = g.standard_normal((m, n))
    return ((U @ V / 8.0 + 0.05 * Z) / np.sqrt(max(m, n))).astype(np.float32)


def vocab_gradient(vocab: int, d: int, seed: int, tokens: int = 12288, zipf_a: float = 1.1) -> np.ndarray:
    """Row-sparse embedding gradient: token ids ~ Zipf(1.1) truncated to the
    vocabulary; each occurrence adds an N(0, 0.01^2)^d row (config 4)."""
    g = rng(seed)
    ids = g.zipf(zipf_a, size=4 * tokens)
    ids = ids[ids <= vocab][:tokens] - 1
    G = np.zeros((vocab, d), np.float64)
    np.add.at(G, ids, g.standard_normal((ids.size, d)) * 0.01)
    return G.astype(np.float32)


def wishart(n: int, seed: int, k: int | None = None) -> np.ndarray:
    """Rank-deficient PSD statistic fl32(W W^T), W in R^{n x k}, k = n/2 by default
    (the "very large condition numbers" of P:211-214 / Fig. 2)."""
    k = max(1, n // 2) if k is None else k
    W = rng(seed).standard_normal((n, k))
    S = W @ W.T
    return ((S + S.T) * 0.5).astype(np.float32)  # exactly symmetric, like every statistic


def spectrum(n: int, seed: int, decades: float = 8.0) -> np.ndarray:
    """fl32(Q diag(10^{-decades*j/(n-1)}) Q^T), Q orthogonal (Householder QR of a Gaussian)."""
    g = rng(seed)
    Q, R = np.linalg.qr(g.standard_normal((n, n)))
    Q = Q * np.sign(np.diag(R))
    lam = 10.0 ** (-decades * np.arange(n) / max(1, n - 1))
    S = (Q * lam) @ Q.T
    return ((S + S.T) * 0.5).astype(np.float32)


def psd_batch(n: int, count: int, seed: int, kind: str = "mixed") -> np.ndarray:
    """(count, n, n) fp32 batch: 'wishart', 'spectrum' or 'mixed' (alternating)."""
    out = np.empty((count, n, n), np.float32)
    for i in range(count):
        use_w = kind == "wishart" or (kind == "mixed" and i % 2 == 0)
        out[i] = wishart(n, seed * 1000 + i) if use_w else spectrum(n, seed * 1000 + i)
    return out


# ------------------------------------------------------------- device (torch)

def torch_generator(seed: int, device):
    import torch
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    return gen


def wishart_batch_device(n: int, count: int, seed: int, device, k: int | None = None, chunk: int = 32):
    """Device (count, n, n) fp32 batch of fl32(W W^T), W ~ N(0,1)^{n x k} drawn
    in fp64 on the device (input generation only -- not the hot path)."""
    import torch
    k = max(1, n // 2) if k is None else k
    gen = torch_generator(seed, device)
    out = torch.empty((count, n, n), dtype=torch.float32, device=device)
    for s in range(0, count, chunk):
        e = min(count, s + chunk)
        W = torch.randn((e - s, n, k), generator=gen, device=device, dtype=torch.float64)
        S = torch.bmm(W, W.transpose(1, 2))
        out[s:e] = ((S + S.transpose(1, 2)) * 0.5).to(torch.float32)
    return out


def lowrank_gradient_device(m: int, n: int, seed: int, device, rank: int = 64):
    import torch
    gen = torch_generator(seed, device)
    U = torch.randn((m, rank), generator=gen, device=device, dtype=torch.float32)
    V = torch.randn((rank, n), generator=gen, device=device, dtype=torch.float32)
    Z = torch.randn((m, n), generator=gen, device=device, dtype=torch.float32)
    return ((U @ V) / 8.0 + 0.05 * Z) / float(np.sqrt(max(m, n)))


def vocab_gradient_device(vocab: int, d: int, seed: int, device, tokens: int = 12288):
    import torch
    return torch.from_numpy(vocab_gradient(vocab, d, seed, tokens)).to(device)
