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


def test_bench_globals_resolve():
    path = os.path.join(REPO, "bench.py")
    spec = importlib.util.spec_from_file_location("bench_static", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
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
