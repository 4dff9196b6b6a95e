"""The reference scheduler API, imported -- not forked.

North star: "The reference's Python policy/scheduler API in pkg/src is kept so
the engine is a drop-in for that path".  The engine therefore plugs into the
real `ecot_sched` package (`/root/reference/pkg/src/ecot_sched`): its trace
types, `GenerationBackend` protocol, `BackendError` hierarchy, runners,
`CachedTrace` and batching accounting are used as they are, and engine
errors are `ecot_sched.backends.BackendError` subclasses so the reference
runners' failure policies (`schedulers.py:411-434`, `:481-483`, `:510-517`)
catch them.

Resolution order: an importable `ecot_sched` (pip-installed), else the
repo-local install `baseline/_ref` (`pip install --target baseline/_ref` of
the reference; it travels with the repo to the GPU box), else the reference
source tree.  There is no fallback copy: if none exists the import fails.
"""

from __future__ import annotations

import os
import sys
import tempfile
from pathlib import Path

_REPO = Path(__file__).resolve().parents[1]
_CANDIDATES = (_REPO / "baseline" / "_ref", Path("/root/reference/pkg/src"))

# numba (the reference's accounting kernels) caches next to the sources;
# the reference tree may be read-only
os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "fastecot_numba_cache"))

try:
    import ecot_sched  # noqa: F401
except ImportError:
    for _c in _CANDIDATES:
        if (_c / "ecot_sched" / "__init__.py").exists():
            sys.path.append(str(_c))
            break
    try:
        import ecot_sched  # noqa: F401
    except ImportError as exc:  # pragma: no cover - environment error
        raise ImportError(
            "the reference scheduler API `ecot_sched` is required (pip install the reference "
            f"package, or install it into {_CANDIDATES[0]})") from exc

from ecot_sched import backends, batching, experiments, schedulers, trace  # noqa: E402,F401

REFERENCE_PATH = Path(ecot_sched.__file__).resolve().parent
