"""pytest plugin: ``import scatterconv`` resolves to the B200 drop-in.

Loaded with ``-p ref_alias`` when the reference's own test modules
(staged unchanged by ``oracle/fetch_ref_tests.py``) run against this
package.  Every module the reference tests import maps onto the drop-in
module that replaces it (pkg/src/scatterconv/*.py → paper_2401_01607_b200/*):

  scatterconv            → paper_2401_01607_b200 (same __all__ names)
  scatterconv.core       → core          scatterconv.engine   → engine
  scatterconv._kernels   → _kernels      scatterconv.bench    → sweeps
  scatterconv.cli        → __main__      scatterconv.quantize → fixed_point
  scatterconv.wavio      → wav
"""

from __future__ import annotations

import importlib
import pathlib
import sys

REPO = pathlib.Path(__file__).resolve().parent.parent
if str(REPO) not in sys.path:
    sys.path.insert(0, str(REPO))

PKG = "paper_2401_01607_b200"
ALIASES = {
    "scatterconv": PKG,
    "scatterconv.core": f"{PKG}.core",
    "scatterconv.engine": f"{PKG}.engine",
    "scatterconv._kernels": f"{PKG}._kernels",
    "scatterconv.bench": f"{PKG}.sweeps",
    "scatterconv.cli": f"{PKG}.__main__",
    "scatterconv.quantize": f"{PKG}.fixed_point",
    "scatterconv.wavio": f"{PKG}.wav",
}


def install() -> None:
    for alias, real in ALIASES.items():
        mod = importlib.import_module(real)
        sys.modules[alias] = mod
        # attribute access (scatterconv.core) as after a real submodule
        # import; a name the package already binds wins, as in the
        # reference (scatterconv.quantize is the function there too)
        if "." in alias and not hasattr(sys.modules["scatterconv"], alias.rsplit(".", 1)[1]):
            setattr(sys.modules["scatterconv"], alias.rsplit(".", 1)[1], mod)


install()
