"""Convenience driver over the C ABI: generate a configured synthetic graph on
the device, build the sketches, select seeds.  Argument marshalling only."""
from __future__ import annotations

from .binding import (PACIM_GEN_ER, PACIM_GEN_GRID, PACIM_GEN_RMAT, PACIM_P_CONST, PACIM_P_WIC,
                      PACIM_P_UNIFORM, pacim_threshold_uniform,
                      Context, pacim_threshold_from_p)


def model_of(cfg: dict) -> tuple[int, int]:
    """(pmodel, t32) of a config dict (see inputs.CONFIGS)."""
    if cfg["pmodel"] == PACIM_P_WIC:
        return PACIM_P_WIC, 0
    if cfg["pmodel"] == PACIM_P_UNIFORM:  # R19: p ~ U(lo, hi) per edge
        return PACIM_P_UNIFORM, pacim_threshold_uniform(*cfg["p_range"])
    return PACIM_P_CONST, pacim_threshold_from_p(cfg["p"])


def center_a32_of(cfg: dict) -> int:
    a = cfg.get("alpha")
    if a is None or a >= 1.0:
        return 1 << 32
    return int(a * 4294967296.0)


def gen_params(cfg: dict) -> tuple[int, list[int]]:
    if cfg["gen"] == 0:
        return PACIM_GEN_ER, [cfg["n"], cfg["m"]]
    if cfg["gen"] == 1:
        ta, tab, tabc = cfg["rmat_t"]
        return PACIM_GEN_RMAT, [cfg["scale"], cfg["ef"], ta, tab, tabc, cfg["permute"]]
    if cfg["gen"] == 2:
        return PACIM_GEN_GRID, [cfg["W"], cfg["H"], cfg["diag_t"]]
    raise ValueError(cfg["gen"])


def generate(ctx: Context, cfg: dict):
    kind, params = gen_params(cfg)
    pm, t32 = model_of(cfg)
    ctx.pacim_generate_graph(kind, params, cfg["gen_seed"], pm, t32)
    return ctx.pacim_graph_info()


def run(ctx: Context, cfg: dict, k: int | None = None):
    """build + select on an already loaded graph; returns (seeds, gain_num, sigma_num, sigma)."""
    ctx.pacim_build_sketches(cfg["R"], cfg["hash_seed"], center_a32_of(cfg))
    return ctx.pacim_select_seeds(k or cfg["k"])
