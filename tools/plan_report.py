"""Print the device planner's waves/passes for a config (host only, no GPU).
usage: python tools/plan_report.py c5 --batch 1024 --mode shared --kind 1"""
import argparse
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1202_3777_b200 import _lib, synth  # noqa: E402
from paper_1202_3777_b200._lib import i32, ptr  # noqa: E402


def plan_handle(tree, dtype):
    cards = i32(tree.cards)
    c_off, c_vars = [0], []
    for c in tree.cliques:
        c_vars += list(c.scope.ids)
        c_off.append(len(c_vars))
    s_edge, s_off, s_vars = [], [0], []
    for s in tree.separators:
        s_edge += list(s.edge)
        s_vars += list(s.scope.ids)
        s_off.append(len(s_vars))
    arrs = [i32(x) for x in (c_off, c_vars, s_edge or [0], s_off, s_vars or [0], tree.roots)]
    h = C.c_void_p()
    _lib.check(_lib.lib().jt_plan_create(len(cards), ptr(cards, C.c_int32), len(tree.cliques), ptr(arrs[0], C.c_int32),
                                         ptr(arrs[1], C.c_int32), len(tree.separators), ptr(arrs[2], C.c_int32),
                                         ptr(arrs[3], C.c_int32), ptr(arrs[4], C.c_int32), len(tree.roots),
                                         ptr(arrs[5], C.c_int32), 0 if dtype == "f32" else 1, 0, C.byref(h)))
    return h, arrs


def report(name, batch=1, mode="materialized", kind=0, dtype="f32", occ=2):
    tree, _ = synth.make_config(name)
    h, _keep = plan_handle(tree, dtype)
    buf = C.create_string_buffer(1 << 22)
    m = 1 if mode == "shared" else 0
    _lib.check(_lib.lib().jt_debug_plan(h, batch, m, kind, 148, occ, buf, len(buf)))
    _lib.lib().jt_plan_destroy(h)
    return buf.value.decode()


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--mode", default="materialized")
    ap.add_argument("--kind", type=int, default=0)
    ap.add_argument("--dtype", default="f32")
    a = ap.parse_args()
    print(report(a.config, a.batch, a.mode, a.kind, a.dtype))
