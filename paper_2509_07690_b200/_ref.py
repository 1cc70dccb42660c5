"""Locate and import the reference package's shipped host code (``polylu``).

The north star keeps preprocessing as the reference's own host code:
``polylu._matching.max_weight_match`` (static pivoting + scaling,
``pkg/src/polylu/_matching.py:169``), ``polylu._amd.amd_permutation``
(``_amd.py:334``), the input type ``polylu.matrix.SparseMatrixCSR``
(``matrix.py:30``), ``polylu.config`` (``SolverConfig``/``KernelMode``) and the
exception hierarchy ``polylu.errors``.  Re-exporting the reference's own classes
makes this package a drop-in: user code catching ``polylu.errors.PatternMismatch``
keeps working.

Search order: an already importable ``polylu``; ``$POLYLU_PATH``;
``<repo>/baseline/_ref`` (the offline ``pip install --target`` of the reference,
which travels to the GPU box); ``/root/reference/pkg/src`` (this container only).
"""

from __future__ import annotations

import importlib
import os
import sys
import tempfile

_REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# numba's cache=True writes next to the module; never into the read-only tree.
os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "hylu_numba_cache"))


def _candidates():
    env = os.environ.get("POLYLU_PATH")
    if env:
        yield env
    yield os.path.join(_REPO, "baseline", "_ref")
    yield "/root/reference/pkg/src"


def _import_polylu():
    try:
        return importlib.import_module("polylu.matrix")
    except ImportError:
        pass
    for path in _candidates():
        if os.path.isdir(os.path.join(path, "polylu")):
            if path not in sys.path:
                sys.path.append(path)
            sys.dont_write_bytecode = True
            try:
                return importlib.import_module("polylu.matrix")
            except ImportError:
                sys.path.remove(path)
    raise ImportError(
        "reference host package 'polylu' not found; install it with "
        "`pip install --no-index --no-deps --target baseline/_ref <copy of /root/reference/pkg>`"
    )


matrix = _import_polylu()
matching = importlib.import_module("polylu._matching")
amd = importlib.import_module("polylu._amd")
config = importlib.import_module("polylu.config")
errors = importlib.import_module("polylu.errors")

SparseMatrixCSR = matrix.SparseMatrixCSR
SolverConfig = config.SolverConfig
KernelMode = config.KernelMode
