"""Find a message whose batched device result differs from the oracle (debug).
usage: python tools/own_debug.py c4M f64 512"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import jtref  # noqa: E402  (checker only)
from paper_1202_3777_b200 import _lib, synth  # noqa: E402
from paper_1202_3777_b200.propagate import plan_for  # noqa: E402
from paper_1202_3777_b200._lib import ptr  # noqa: E402

name, dt, B = sys.argv[1], sys.argv[2], int(sys.argv[3])
tree, tables = synth.make_config(name)
L = _lib.lib()
plan = plan_for(tree, dt)
h = C.c_void_p()
_lib.check(L.jt_state_create(plan.handle, B, 0, C.byref(h)))
cat = np.concatenate(tables)
_lib.check(L.jt_state_load(h, -1, ptr(cat, C.c_double), None))
csz = [c.scope.size for c in tree.cliques]
ssz = [s.scope.size for s in tree.separators]
hc = np.empty(sum(csz)); hs = np.empty(max(1, sum(ssz)))
co = np.concatenate([[0], np.cumsum(csz)]); so = np.concatenate([[0], np.cumsum(ssz)])
bad = 0
mc = [np.asarray(t, float).copy() for t in tables]
ms = [np.ones(n) for n in ssz]
for s in tree.separators[:300]:
    for (a, b) in (s.edge, s.edge[::-1]):
        mu_s = jtref.build_mapping_table(tree.cliques[a].scope.ids, tree.cliques[a].scope.cards, s.scope.ids)
        mu_t = jtref.build_mapping_table(tree.cliques[b].scope.ids, tree.cliques[b].scope.cards, s.scope.ids)
        jtref.pass_block(mc[a], mc[b], ms[s.id], mu_s, mu_t, 0, len(ms[s.id]))
        _lib.check(L.jt_message(h, a, b, s.id, None))
        _lib.check(L.jt_sync_error(h))
        L.jt_state_store(h, B - 1, ptr(hc, C.c_double), ptr(hs, C.c_double))
        gs, gt = hs[so[s.id]:so[s.id + 1]], hc[co[b]:co[b + 1]]
        e1 = np.max(np.abs(gs - ms[s.id]) / np.maximum(np.abs(ms[s.id]), 1e-300))
        e2 = np.max(np.abs(gt - mc[b]) / np.maximum(np.abs(mc[b]), 1e-300))
        if e1 > 1e-10 or e2 > 1e-10:
            bad += 1
            print("BAD msg", a, "->", b, "sep", s.id, "sep err %.2e tgt err %.2e" % (e1, e2),
                  "src", tree.cliques[a].scope.ids, tree.cliques[a].scope.cards, "sep", s.scope.ids,
                  "tgt", tree.cliques[b].scope.ids, tree.cliques[b].scope.cards, flush=True)
            # resync the mirror with the device to keep checking later messages
            ms[s.id] = gs.copy()
            mc[b] = gt.copy()
            if bad > 6:
                sys.exit(0)
print("done bad", bad)
