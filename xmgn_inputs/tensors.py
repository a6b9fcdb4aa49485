"""Counter-based synthetic values, identical on CPU and GPU.

Every value is a pure function of (seed, tensor id, row, col) through a 32-bit
murmur3-finaliser chain evaluated in int64 torch arithmetic without overflow,
mapped to a uniform u in (0, 1), scaled in FP64, cast to FP32 and rounded to a
BF16-representable value (round-to-nearest-even).  Because every step is exact
integer arithmetic or a correctly rounded IEEE operation, the same bits come out
on any device, so a partition's local rows (hashed by GLOBAL node / edge id)
equal the full graph's rows.

Seeds: params 1, h0 2, e0 3, g 4.  Distributions: W, b ~
U(+-1/sqrt(fan_in)); gamma = 1 + 0.1*U(+-sqrt3); beta = 0.1*U(+-sqrt3);
h0, e0, g ~ U(+-sqrt3) (unit variance).

``param_layout`` restates the flat FP32 parameter layout of the C-ABI
 so the generator can place gamma/beta values; the oracle and the
library each implement the layout independently.
"""
import math
import torch

M32 = 0xFFFFFFFF
SEED_PARAMS, SEED_H0, SEED_E0, SEED_G = 1, 2, 3, 4


def _mul32(h, c):
    """(h * c) mod 2^32 for int64 tensors 0 <= h < 2^32 without int64 overflow."""
    hi = h >> 16
    lo = h & 0xFFFF
    return ((((hi * c) & 0xFFFF) << 16) + lo * c) & M32


def _fmix32(h):
    h = h ^ (h >> 16)
    h = _mul32(h, 0x85EBCA6B)
    h = h ^ (h >> 13)
    h = _mul32(h, 0xC2B2AE35)
    return h ^ (h >> 16)


def _fmix32_int(h):
    h &= M32
    h ^= h >> 16
    h = (h * 0x85EBCA6B) & M32
    h ^= h >> 13
    h = (h * 0xC2B2AE35) & M32
    return h ^ (h >> 16)


def uniform(seed, tensor_id, rows, ncols, device="cpu"):
    """u in (0,1), float64 tensor [len(rows), ncols]."""
    rows = torch.as_tensor(rows, dtype=torch.int64, device=device)
    base = _fmix32_int(seed * 0x9E3779B1 + tensor_id)
    x = _fmix32((rows & M32) ^ base)[:, None]
    cols = torch.arange(ncols, dtype=torch.int64, device=device)[None, :]
    x = _fmix32((x + cols * 0x27D4EB2F) & M32)
    return (x.to(torch.float64) + 0.5) * (1.0 / 4294967296.0)


def bf16_exact(x64):
    """FP64 -> FP32 -> BF16 (RNE) -> FP32."""
    return x64.to(torch.float32).to(torch.bfloat16).to(torch.float32)


def sym_uniform(seed, tensor_id, rows, ncols, scale, device="cpu", chunk=1 << 20):
    """BF16-exact FP32 values scale*(2u-1), generated in row chunks."""
    rows = torch.as_tensor(rows, dtype=torch.int64, device=device)
    out = torch.empty((len(rows), ncols), dtype=torch.float32, device=device)
    step = max(1, chunk // max(ncols, 1))
    for r0 in range(0, len(rows), step):
        u = uniform(seed, tensor_id, rows[r0:r0 + step], ncols, device)
        out[r0:r0 + step] = bf16_exact(scale * (2.0 * u - 1.0))
    return out


SQRT3 = math.sqrt(3.0)


def node_features(gids, H, device="cpu"):
    return sym_uniform(SEED_H0, 0, gids, H, SQRT3, device)


def edge_features(gids, H, device="cpu"):
    return sym_uniform(SEED_E0, 0, gids, H, SQRT3, device)


def upstream_grad(gids, H, device="cpu"):
    return sym_uniform(SEED_G, 0, gids, H, SQRT3, device)


def param_layout(H, L, m=2):
    """List of (name, layer, block, slot, offset, shape, fan_in) in ABI order.

    Per layer: edge block W1[3H,H] (row blocks e, h_src, h_dst), b1, then for
    j=2..m+1 Wj[H,H], bj, then gamma, beta; node block W1[2H,H] (h, agg), b1,
    Wj, bj, gamma, beta.  y = x W + b with W stored [in, out].
    """
    out, off = [], 0
    for l in range(L):
        for blk, kin in ((0, 3 * H), (1, 2 * H)):
            slot = 0
            fan = kin
            for j in range(m + 1):
                kin_j = kin if j == 0 else H
                out.append((f"W{j+1}", l, blk, slot, off, (kin_j, H), kin_j)); off += kin_j * H; slot += 1
                out.append((f"b{j+1}", l, blk, slot, off, (H,), kin_j)); off += H; slot += 1
                fan = kin_j
            out.append(("gamma", l, blk, slot, off, (H,), fan)); off += H; slot += 1
            out.append(("beta", l, blk, slot, off, (H,), fan)); off += H; slot += 1
    return out, off


def param_count(H, L, m=2):
    return L * ((5 + 2 * m) * H * H + (2 * m + 6) * H)


def params(H, L, m=2, device="cpu"):
    lay, n = param_layout(H, L, m)
    assert n == param_count(H, L, m)
    p = torch.empty(n, dtype=torch.float32, device=device)
    for name, l, blk, slot, off, shape, fan in lay:
        tid = (l * 2 + blk) * 16 + slot
        rows = torch.arange(shape[0], device=device)
        ncol = shape[1] if len(shape) == 2 else 1
        if name == "gamma":
            v = 1.0 + sym_uniform(SEED_PARAMS, tid, rows, ncol, 0.1 * SQRT3, device)
            v = v.to(torch.bfloat16).to(torch.float32)
        elif name == "beta":
            v = sym_uniform(SEED_PARAMS, tid, rows, ncol, 0.1 * SQRT3, device)
        else:
            v = sym_uniform(SEED_PARAMS, tid, rows, ncol, 1.0 / math.sqrt(fan), device)
        p[off:off + v.numel()] = v.reshape(-1)
    return p


# ---------------------------------------------------------------- model inputs (NEXT-1)
SEED_TARGETS, SEED_IO = 5, 6
F_NODE, F_EDGE, D_OUT = 24, 4, 4   # PAPER.md:234 (24 inputs), :161 (4 edge features), :217 (p, tau)


def io_param_layout(H, m=2, fn=F_NODE, fe=F_EDGE, d=D_OUT):
    """(name, block, slot, offset, shape, fan_in) of the encoder / decoder parameters in
    the C-ABI order (include/xmgn.h): node encoder, edge encoder (W1, b1, ..., gamma,
    beta), decoder (W1, b1, ..., W_{m+1} [H x d], b_{m+1} [d])."""
    out, off = [], 0
    for blk, fin in ((0, fn), (1, fe)):
        slot = 0
        for j in range(m + 1):
            kin = fin if j == 0 else H
            out.append((f"W{j+1}", blk, slot, off, (kin, H), kin)); off += kin * H; slot += 1
            out.append((f"b{j+1}", blk, slot, off, (H,), kin)); off += H; slot += 1
        out.append(("gamma", blk, slot, off, (H,), H)); off += H; slot += 1
        out.append(("beta", blk, slot, off, (H,), H)); off += H; slot += 1
    slot = 0
    for j in range(m + 1):
        nout = d if j == m else H
        out.append((f"W{j+1}", 2, slot, off, (H, nout), H)); off += H * nout; slot += 1
        out.append((f"b{j+1}", 2, slot, off, (nout,), H)); off += nout; slot += 1
    return out, off


def io_params(H, m=2, device="cpu"):
    lay, n = io_param_layout(H, m)
    p = torch.empty(n, dtype=torch.float32, device=device)
    for name, blk, slot, off, shape, fan in lay:
        tid = blk * 16 + slot
        rows = torch.arange(shape[0], device=device)
        ncol = shape[1] if len(shape) == 2 else 1
        if name == "gamma":
            v = (1.0 + sym_uniform(SEED_IO, tid, rows, ncol, 0.1 * SQRT3, device)).to(torch.bfloat16).to(torch.float32)
        elif name == "beta":
            v = sym_uniform(SEED_IO, tid, rows, ncol, 0.1 * SQRT3, device)
        else:
            v = sym_uniform(SEED_IO, tid, rows, ncol, 1.0 / math.sqrt(fan), device)
        p[off:off + v.numel()] = v.reshape(-1)
    return p


def targets(gids, device="cpu"):
    """Synthetic z-scored targets (p, tau_x, tau_y, tau_z) ~ U(+-sqrt3) per node."""
    return sym_uniform(SEED_TARGETS, 0, gids, D_OUT, SQRT3, device)
