"""B200-native core-Hamiltonian path of arXiv 1408.3839 (latham reference, proj/core).

``system``  LatticeSystem + seeded BASELINE configs (no GPU needed)
``native``  ctypes loader of the sm_100a engine (_lib/liblatham_b200.so)
``api``     reference-shaped API (assemble_box/assemble_periodic/combine/solve_*)
``dist``    k-point sharding over torch.distributed ranks
"""
from .system import CONFIG_NAMES, LatticeSystem, config_periodic, make_config  # noqa: F401

__all__ = ["LatticeSystem", "make_config", "config_periodic", "CONFIG_NAMES"]
