"""B200-native rk-Rotor chain solver (the hot path of Rockmate, arXiv 2307.01236).

The DP of /root/reference/proj/include/remat/chain_dp.hpp runs as sm_100a CUDA
kernels in ``librkr.so`` (C ABI: include/rkr.h).  ``rotor`` mirrors the
reference's ``remat`` API for Python callers; ``menu`` holds option menus and
the synthetic chain generator.
"""
from .menu import BlockOption, Menu, config_menu, synthetic_menu, tiny_chain_menu  # noqa: F401
from .rotor import (  # noqa: F401
    K_INF_TIME,
    Chain,
    ChainSolution,
    DeviceError,
    DpArg,
    DpTable,
    InfeasibleBudget,
    ScheduleOp,
    ValidationError,
    build_schedule_rec,
    quantize,
    solve_chain,
    to_units,
)
