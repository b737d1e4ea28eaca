"""B200-native trijoin: filter-and-refine spatial joins over triangulated polyhedra.

Drop-in for the reference's Python package ``trijoin`` (proj/python/trijoin/__init__.py)
on the join path: ``join(r, s="", **kwargs)`` returns ``{"records": [...], "stats": {...}}``
with the same keyword arguments (type, tau, k, filter_chunk, refine_chunk, lods, pipeline,
workers, seed, exact). The work runs on B200 GPUs through ``libtrijoin_b200.so`` (C-ABI in
include/tj_capi.h); there is no CPU fallback — importing fails loudly if the compiled
extension is missing, and joining fails loudly without a B200.

``oracle(r, s="", **kwargs)`` is the reference's exhaustive exact join (``trijoin.oracle``),
here on the GPU. Dataset generation / preprocessing are offline tooling in the reference and
are out of scope.
"""

import json
import os

_HERE = os.path.dirname(os.path.abspath(__file__))

try:
    from . import _core  # noqa: F401  (loads libtrijoin_b200.so via rpath)
except ImportError as exc:  # pragma: no cover - exercised only on a broken install
    raise ImportError(
        "paper_2604_19982_b200._core is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
        f"or `make -C {os.path.join(_HERE, 'csrc')}` ({exc})"
    ) from exc

from ._core import EngineError, IndexError, Resident, join_datasets, load_dataset, replicate_index  # noqa: E402

__all__ = [
    "join",
    "oracle",
    "join_datasets",
    "load_dataset",
    "replicate_index",
    "Resident",
    "EngineError",
    "IndexError",
    "LIB_PATH",
]

LIB_PATH = os.path.join(_HERE, "libtrijoin_b200.so")


def join(r, s="", **kwargs):
    """Run a join between two index files (self-join when ``s`` is empty).

    Returns ``{"records": [(r, s, lb, ub, stage, rank), ...], "stats": dict}`` exactly like
    the reference's ``trijoin.join``.
    """
    records, stats = _core.join(r, s, **kwargs)
    return {"records": records, "stats": json.loads(stats)}


def oracle(r, s="", **kwargs):
    """Exact reference join over the original-resolution geometry (reference ``trijoin.oracle``),
    evaluated on the GPU. Same result shape as :func:`join`; accepts type, tau, k, workers, seed.
    """
    records, stats = _core.oracle(r, s, **kwargs)
    return {"records": records, "stats": json.loads(stats)}
