"""Drop-in for the reference Python module ``hbp`` (bindings/py_hbp.cpp).

    from paper_2503_07680_b200 import hbp
    plan = hbp.build_plan(hbp.SampleSet(lengths), groups, device_count=8)

Same names, argument names, defaults and exception mapping as the
reference; every plan-level call runs on the B200 engine (libhbp_b200.so)
through the C++ façade (libhbp_facade.so). Importing fails when the native
libraries are missing -- there is no Python fallback.
"""
from ._hbp import *  # noqa: F401,F403
from ._hbp import InfeasibleError, IoError, ValidationError  # noqa: F401
