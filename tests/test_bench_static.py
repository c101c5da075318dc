"""bench.py is only executed end to end on a GPU box: catch undefined globals here.

Every LOAD_GLOBAL in bench.py (nested functions included) must resolve to a
module-level name or a builtin -- a stale local (e.g. a timer read in a
function that never set it) compiles to a global lookup and would only fail
at the driver's round-end run.
"""

import builtins
import dis
import importlib.util
import os
import types

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _codes(co):
    yield co
    for c in co.co_consts:
        if isinstance(c, types.CodeType):
            yield from _codes(c)


import importlib

import pytest


def _load(rel):
    path = os.path.join(REPO, rel)
    if rel.endswith("session.py"):
        ref = os.path.join(REPO, "baseline", "_ref")
        if not os.path.isdir(os.path.join(ref, "diffusekit")):
            pytest.skip("reference not installed (baseline/_ref)")
        import sys

        if ref not in sys.path:
            sys.path.append(ref)
    if rel.startswith("paper_2406_18109_b200/"):
        return path, importlib.import_module(rel[:-3].replace("/", "."))
    spec = importlib.util.spec_from_file_location(rel.replace("/", "_")[:-3] + "_static", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return path, mod


@pytest.mark.parametrize("rel", ["bench.py", "__graft_entry__.py", "paper_2406_18109_b200/executor.py",
                                 "paper_2406_18109_b200/streaming.py", "paper_2406_18109_b200/session.py",
                                 "paper_2406_18109_b200/runtime.py", "tools/host_overhead.py"])
def test_globals_resolve(rel):
    path, mod = _load(rel)
    src = open(path).read()
    top = compile(src, path, "exec")
    missing = set()
    for co in _codes(top):
        if co is top:
            continue
        for ins in dis.get_instructions(co):
            if ins.opname == "LOAD_GLOBAL":
                name = ins.argval
                if not hasattr(mod, name) and not hasattr(builtins, name):
                    missing.add((co.co_name, name))
    assert not missing, sorted(missing)
