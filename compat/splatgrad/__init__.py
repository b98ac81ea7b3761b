"""Import shim: `splatgrad` (the reference package's name) backed by the
B200 build.  Put `compat/` first on PYTHONPATH and unmodified callers of
the reference -- `import splatgrad as sg; sg.render(...)` -- run on the GPU
path (paper_2312_02121_b200; every name of the reference's
sg/__init__.py:64-119).  Submodules the reference's own tests import by
path (raster_forward, projection, cli) are mapped too.  This is glue, not
the reference: no reference code lives here.
"""

import paper_2312_02121_b200 as _b200
from paper_2312_02121_b200 import *  # noqa: F401,F403

__all__ = list(_b200.__all__)
__version__ = _b200.__version__
