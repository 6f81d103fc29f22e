"""Drop-in import name: ``import lidarsplat`` resolves to the B200 package.

Aliases every submodule of paper_2502_11618_b200 under ``lidarsplat.*`` so code
written against the reference (``from lidarsplat.render import candidates``,
``from lidarsplat._kernels import get_backend`` ...) runs unchanged.
"""

import importlib
import pkgutil
import sys

import paper_2502_11618_b200 as _impl

for _m in pkgutil.walk_packages(_impl.__path__, _impl.__name__ + "."):
    if _m.name.endswith(".build"):
        continue
    try:
        sys.modules["lidarsplat" + _m.name[len(_impl.__name__):]] = importlib.import_module(_m.name)
    except ImportError:  # optional pieces (none today)
        pass

sys.modules[__name__] = _impl
