"""B200-native Galerkin surface multigrid (arXiv 2104.13755): C-ABI library
libmg (include/mg.h, csrc/) with a thin ctypes binding (mg.py)."""
from . import mg  # noqa: F401
from .mg import Solver, MGError  # noqa: F401

__all__ = ["mg", "Solver", "MGError"]
