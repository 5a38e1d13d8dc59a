"""TEST INFRASTRUCTURE ONLY -- imports the read-only reference package in place.

The reference package ``lfsrcycles`` (/root/reference/pkg/src/lfsrcycles) does not
import as shipped: ``__init__.py:26`` imports a ``stats`` module that does not exist
(SURVEY.md §0, Appendix D.1).  This shim registers a bare package object whose
``__path__`` points at the reference sources, so the submodules (cipher, bitslice,
pipeline, records, oracle) import normally without executing ``__init__.py``.

Only ``oracle/gen_golden.py`` and CPU tests that explicitly skip when the reference
is absent use this.  /root/reference does not exist on the GPU box; nothing in the
GPU tests, ``smoke()`` or ``bench.py`` may import this module.
"""

from __future__ import annotations

import os
import sys
import types

REF_SRC = os.environ.get("LFSR_REFERENCE_SRC", "/root/reference/pkg/src/lfsrcycles")


def available() -> bool:
    return os.path.isfile(os.path.join(REF_SRC, "cipher.py"))


def load():
    """Return a namespace with the reference submodules (cipher, bitslice, ...)."""
    if not available():
        raise ImportError(f"reference sources not found at {REF_SRC}")
    sys.dont_write_bytecode = True  # the tree is read-only
    if "lfsrcycles" not in sys.modules:
        pkg = types.ModuleType("lfsrcycles")
        pkg.__path__ = [REF_SRC]
        sys.modules["lfsrcycles"] = pkg
    import importlib

    ns = types.SimpleNamespace()
    for name in ("cipher", "bitslice", "pipeline", "records", "oracle", "extsort", "reduce"):
        setattr(ns, name, importlib.import_module(f"lfsrcycles.{name}"))
    return ns
