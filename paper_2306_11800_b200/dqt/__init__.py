"""Drop-in for the reference Python module ``dqt`` (B200 engine underneath).

``from paper_2306_11800_b200 import dqt`` exposes the same names as the
reference's ``dqt`` package (bindings/py_module.cpp); put
``paper_2306_11800_b200`` on ``sys.path`` to keep ``import dqt`` unchanged.
"""
from ._dqt import *  # noqa: F401,F403
from ._dqt import __doc__  # noqa: F401
