"""pytest plugin: run the reference package's OWN test suite with this
repo's B200 engine hot-swapped into it (paper_2406_18820_b200.hotswap).

    rm -rf baseline/_ref_tests && cp -r /root/reference/pkg/tests baseline/_ref_tests  # git-ignored
    PYTHONPATH=baseline/_ref:.:tools python -m pytest baseline/_ref_tests -p ref_suite_plugin -q

The swap happens in pytest_configure, before any test module runs
``from ucp import convert, load, ...``. ``ucp.parallel.extract_fragment`` and
``ucp.oracle`` stay the reference's: the suite uses them as expected values.
The terminal summary reports how many calls each swapped entry point served,
so a pass cannot come from the reference's own code path silently.
"""

from __future__ import annotations

import collections
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CALLS: collections.Counter = collections.Counter()


def pytest_configure(config):
    ref = os.path.join(ROOT, "baseline", "_ref")
    for p in (ROOT, ref):
        if p not in sys.path:
            sys.path.insert(0, p)
    import ucp

    if os.path.dirname(os.path.dirname(ucp.__file__)) != ref:
        raise RuntimeError(f"ucp imported from {ucp.__file__}, expected baseline/_ref")
    from paper_2406_18820_b200 import api, hotswap

    for name in ("convert", "load", "resume", "union", "extract_fragment", "ucp_info"):
        fn = getattr(api, name)

        def counted(*a, __fn=fn, __name=name, **k):
            CALLS[__name] += 1
            return __fn(*a, **k)

        setattr(api, name, counted)
    config._ucp_undo = hotswap.install(ucp)


def pytest_unconfigure(config):
    undo = getattr(config, "_ucp_undo", None)
    if undo is not None:
        undo()


def pytest_terminal_summary(terminalreporter):
    from paper_2406_18820_b200 import _native

    lib = _native.LIB_PATH if _native._lib is not None else "(not loaded)"
    terminalreporter.write_line(f"B200 engine calls served under the reference suite: {dict(CALLS)}")
    terminalreporter.write_line(f"native library: {lib}")
