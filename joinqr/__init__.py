"""`joinqr` drop-in shim: the reference's package name, served by the B200 build.

`import joinqr` resolves every hot-path name of the reference
(pkg/src/joinqr/__init__.py:20-62) lazily from paper_2503_23385_b200.
"""

import paper_2503_23385_b200 as _impl

__version__ = _impl.__version__


def __getattr__(name):
    return getattr(_impl, name)


def __dir__():
    return dir(_impl)
