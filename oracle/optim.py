"""FP64 optimiser step (NEXT-2) -- TEST INFRASTRUCTURE ONLY (tests/, bench.py's
reference leg; never the product).

PAPER.md:234 (Sec. V-D): "The Adam optimizer is used with a cosine annealing
learning rate schedule ranging from 1e-3 to 1e-6 ... Gradient clipping with a
threshold of 32", with the readings of SPEC.md:373-381 / 391: global-L2-norm
clipping after cross-partition aggregation, betas 0.9 / 0.999, eps 1e-8, cosine
lr(t) = lr_min + (lr_max - lr_min)(1 + cos(pi t / T)) / 2 with t = 0 at the first
step, and Adam's bias corrections with t + 1 (Kingma & Ba, Algorithm 1).  Each
function is the textbook formula, step by step.  Pins: tests/test_optim.py
(cosine endpoints, the clip example of SPEC.md:380, torch.optim.Adam +
clip_grad_norm_ in float64, multi-step partitioned = full-graph training).
"""
import math

import numpy as np


def cosine_lr(step, total_steps, lr_max=1e-3, lr_min=1e-6):
    t = min(step, total_steps)
    return lr_min + 0.5 * (lr_max - lr_min) * (1.0 + math.cos(math.pi * t / total_steps))


def clip_global_norm(g, clip):
    """g * min(1, clip / (||g||_2 + 1e-6)) and ||g||_2 (the norm before clipping)."""
    norm = math.sqrt(float(np.sum(np.asarray(g, np.float64) ** 2)))
    coef = min(1.0, clip / (norm + 1e-6))
    return g * coef, norm


def adam_step(p, g, m, v, step, total_steps, lr_max=1e-3, lr_min=1e-6, beta1=0.9, beta2=0.999, eps=1e-8,
              clip=32.0, grad_scale=1.0):
    """One step; returns (p, m, v, norm).  Arrays are not modified in place."""
    g = np.asarray(g, np.float64) * grad_scale
    g, norm = clip_global_norm(g, clip)
    m = beta1 * m + (1.0 - beta1) * g
    v = beta2 * v + (1.0 - beta2) * g * g
    m_hat = m / (1.0 - beta1 ** (step + 1))
    v_hat = v / (1.0 - beta2 ** (step + 1))
    lr = cosine_lr(step, total_steps, lr_max, lr_min)
    p = p - lr * m_hat / (np.sqrt(v_hat) + eps)
    return p, m, v, norm
