"""B200-native forward DGT on a nonseparable lattice (shear algorithm, arXiv:1307.4569).

Public API (see ``include/nsdgt.h`` for the C ABI underneath):
    Plan(L, a, M, lam1, lam2, g, dtype="c64"|"c128", ...).execute(f) -> c[W, M, N]
    Plan(..., algorithm="multiwindow")           (the comparison algorithm of Sec. 3.1)
    Plan.execute_host(f_host) -> c_host          (end to end through host buffers)
    lattice_plan(L, a, M, lam1, lam2)            (host-only planner record)

The binding is loaded lazily so that ``python -m paper_1307_4569_b200.build`` works
before the library exists; touching any API name loads ``libnsdgt.so`` or raises.
"""
__all__ = ["Plan", "lattice_plan", "DgtError", "LatticeInfo", "BRANCH_NAMES", "version",
           "DGT_OK", "DGT_EINVAL", "DGT_EILLEGAL_LENGTH", "DGT_ECUDA", "DGT_ECUFFT", "DGT_ENOMEM",
           "DGT_EUNSUPPORTED"]


def __getattr__(name):
    if name in __all__:
        from . import nsdgt as _b
        return getattr(_b, name)
    raise AttributeError(name)
