"""pytest plugin (`-p ref_install_plugin`): route the reference package
through the B200 path BEFORE the reference's own tests import it.

The reference's tests import `fused_sweep`, `assemble_collision`, ... by
value from `axlandau` (e.g. test_kernel.py:8-21), so the patch must be in
place when their modules are imported; `-p` plugins load before any
conftest or test module.  Every patched entry point is wrapped with a call
counter, written at the end of the session to $LB_REF_CALLS (JSON), so the
caller can prove the B200 functions -- not the reference's -- were exercised.
"""

import atexit
import json
import os

import axlandau

import paper_1702_08880_b200 as lb

SAVED = lb.install(axlandau)
CALLS: dict = {}


def _wrap(mod, name):
    fn = getattr(mod, name)
    key = f"{mod.__name__}.{name}"
    CALLS.setdefault(key, 0)

    def counted(*a, **k):
        CALLS[key] += 1
        return fn(*a, **k)

    counted.__wrapped__ = fn
    counted.__name__ = getattr(fn, "__name__", name)
    counted.__doc__ = getattr(fn, "__doc__", None)
    setattr(mod, name, counted)


def _install_counters():
    import importlib

    for (mod_name, nm) in SAVED:
        if mod_name == "@":
            continue
        mod = axlandau if not mod_name else importlib.import_module(f"axlandau.{mod_name}")
        _wrap(mod, nm)


_install_counters()


def pytest_report_header(config):
    return ("axlandau routed through paper_1702_08880_b200 (install): "
            + ", ".join(sorted(CALLS)))


@atexit.register
def _dump():
    out = os.environ.get("LB_REF_CALLS")
    if out:
        with open(out, "w") as fh:
            json.dump(CALLS, fh, indent=1, sort_keys=True)
