"""Synthetic operands exactly as the reference's bench harness makes them.

`SweepConfig` / `build_chain` / `make_operands` restate the recipe of the
reference's `bench.py:45-64,99-115,138-140`: factor seeds from
`SeedSequence(seed).generate_state(2)`, a complete factor whenever a sparsity
is 0, then `init_random` on `make_rng(SeedSequence([seed, 1]).generate_state(1)[0])`
followed by `uniform(-1, 1, (K, N))` on the same generator.  Given the same
config the arrays are bit-identical to what the reference feeds its kernel,
which is what makes output hashes comparable.

Also holds the named layer tables the benchmark uses (VGG19-CIFAR 512-channel
convolutions via im2col).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .generate import LiftChainSpec, generate_ramanujan, make_rng
from .graphs import complete_graph
from .products import RbgpChain
from .rcubs import init_random


@dataclass(frozen=True)
class SweepConfig:
    """One synthetic multiply: factor shapes, sparsity split, column count."""

    config_id: str
    g_o: tuple
    sp_o: float
    g_r: tuple
    g_i: tuple
    sp_i: float
    g_b: tuple
    n_cols: int
    tn: int = 128
    rn: int = 1
    bn: int = 32
    workers: int = 4
    precision: str = "f32"
    runs: int = 5
    warmup: int = 2
    seed: int = 0


def _factor(shape, sparsity, seed):
    if sparsity == 0.0:
        return complete_graph(*shape)
    return generate_ramanujan(LiftChainSpec(shape[0], shape[1], sparsity, rng_seed=seed)).graph


def build_chain(cfg: SweepConfig) -> RbgpChain:
    s_o, s_i = (int(x) for x in np.random.SeedSequence(cfg.seed).generate_state(2))
    return RbgpChain((
        _factor(cfg.g_o, cfg.sp_o, s_o),
        complete_graph(*cfg.g_r),
        _factor(cfg.g_i, cfg.sp_i, s_i),
        complete_graph(*cfg.g_b),
    ))


def make_operands(cfg: SweepConfig, chain: RbgpChain | None = None):
    """(chain, W, I) for a config; W is an RcubsMatrix, I a (K, N) array."""
    chain = build_chain(cfg) if chain is None else chain
    rng = make_rng(np.random.SeedSequence([cfg.seed, 1]).generate_state(1)[0])
    w = init_random(chain, rng, precision=cfg.precision)
    inp = rng.uniform(-1.0, 1.0, size=(w.cols, cfg.n_cols)).astype(w.dtype)
    return chain, w, inp


# Config 1 of BASELINE.json (SURVEY §7 "minimum slice", factorisation C1a).
C1A = SweepConfig("cfg1", (8, 16), 0.5, (2, 1), (32, 32), 0.5, (1, 1), n_cols=1024,
                  precision="f32", seed=0)
# tensor-core-shaped variant of config 1 (C1b): TM = TK = 128, g = 16.
C1B = SweepConfig("cfg1b", (4, 4), 0.5, (4, 1), (8, 8), 0.5, (4, 16), n_cols=1024,
                  precision="f32", seed=0)


def vgg19_cifar_512(sparsity: float = 0.875, batch: int = 256, seed: int = 0):
    """The 512-output-channel convolutions of VGG19-CIFAR as im2col SDMMs.

    (M, K, N) = (C_out, 9 C_in, batch H W): conv9 is 256->512 at 4x4, conv10-12
    512->512 at 4x4, conv13-16 512->512 at 2x2.  The
    factorisation follows the survey's recipe -- tile 128x64, G_r = (4,1),
    G_b = (1,1), G_o = (M/128, K/64) at 50 %, G_i = (32, 64) carrying the rest
    -- so 75 / 87.5 / 93.75 % are G_i at 50 / 75 / 87.5 %.
    """
    sp_i = {0.75: 0.5, 0.875: 0.75, 0.9375: 0.875}[sparsity]
    layers = [("conv9", 512, 2304, batch * 16)]
    layers += [(f"conv{i}", 512, 4608, batch * 16) for i in (10, 11, 12)]
    layers += [(f"conv{i}", 512, 4608, batch * 4) for i in (13, 14, 15, 16)]
    out = []
    for idx, (name, m, k, n) in enumerate(layers):
        out.append(SweepConfig(
            f"vgg19-{name}-sp{sparsity * 100:g}", (m // 128, k // 64), 0.5, (4, 1), (32, 64),
            sp_i, (1, 1), n_cols=n, precision="f32", seed=seed + idx,
        ))
    return out


def vgg19_cifar_512_tc(sparsity: float = 0.875, batch: int = 256, seed: int = 0):
    """Same VGG19-CIFAR layers, tensor-core-friendly factorisation (SURVEY §7 hard part 1).

    Tile 128 x 128 with G_r = (1,1), G_b = (8,8) dense 8x8 element blocks, G_o = (4, K/128)
    at 50 % and G_i = (16,16) carrying the rest: 75 / 87.5 / 93.75 % are G_i at
    50 / 75 / 87.5 %.  Every nonzero run along K is 8 elements (16 bytes of bf16), which
    the tensor-core kernel scatters with 16-byte stores.
    """
    sp_i = {0.75: 0.5, 0.875: 0.75, 0.9375: 0.875}[sparsity]
    layers = [("conv9", 512, 2304, batch * 16)]
    layers += [(f"conv{i}", 512, 4608, batch * 16) for i in (10, 11, 12)]
    layers += [(f"conv{i}", 512, 4608, batch * 4) for i in (13, 14, 15, 16)]
    out = []
    for idx, (name, m, k, n) in enumerate(layers):
        out.append(SweepConfig(
            f"vgg19tc-{name}-sp{sparsity * 100:g}", (m // 128, k // 128), 0.5, (1, 1), (16, 16),
            sp_i, (8, 8), n_cols=n, precision="f32", seed=seed + idx,
        ))
    return out


def vgg19_cifar_512_tc16(sparsity: float = 0.875, batch: int = 256, seed: int = 0):
    """Same VGG19-CIFAR layers with 16 x 16 dense element blocks ("VGG c10 TC").

    Tile 128 x 128 with G_r = (1,1), G_b = (16,16), G_o = (4, K/128) at 50 % and G_i = (8,8)
    carrying the rest: 75 / 87.5 % are G_i at 50 / 75 %.  Blocks of 16 x 16 are whole MMA
    operands, so the product runs on the gathered-block kernel (no densification).
    """
    sp_i = {0.75: 0.5, 0.875: 0.75}[sparsity]
    layers = [("conv9", 512, 2304, batch * 16)]
    layers += [(f"conv{i}", 512, 4608, batch * 16) for i in (10, 11, 12)]
    layers += [(f"conv{i}", 512, 4608, batch * 4) for i in (13, 14, 15, 16)]
    out = []
    for idx, (name, m, k, n) in enumerate(layers):
        out.append(SweepConfig(
            f"vgg19tc16-{name}-sp{sparsity * 100:g}", (m // 128, k // 128), 0.5, (1, 1), (8, 8),
            sp_i, (16, 16), n_cols=n, precision="f32", seed=seed + idx,
        ))
    return out
