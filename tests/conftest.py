import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")
REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libjtb200.so")
    config.addinivalue_line("markers", "reference: needs the reference package at /root/reference")


def have_reference():
    return os.path.isdir(REFERENCE_SRC)


def tree_from_json(doc):
    """Rebuild the exact reference tree (cliques, separators, roots) from a fixture."""
    from paper_1202_3777_b200.tree import Clique, JunctionTree, Scope, Separator

    cards = tuple(doc["cards"])
    cliques = [Clique(i, tuple(m), Scope(tuple(m), tuple(cards[v] for v in m)))
               for i, m in enumerate(doc["cliques"])]
    seps, nbrs = [], [[] for _ in cliques]
    for sid, (edge, members) in enumerate(doc["separators"]):
        seps.append(Separator(sid, tuple(edge), tuple(members),
                              Scope(tuple(members), tuple(cards[v] for v in members))))
        nbrs[edge[0]].append((edge[1], sid))
        nbrs[edge[1]].append((edge[0], sid))
    for l in nbrs:
        l.sort()
    return JunctionTree(cards, cliques, seps, nbrs, list(doc["roots"]),
                        {int(k): v for k, v in doc.get("cpt_assignment", {}).items()})


def load_golden(name):
    with open(os.path.join(GOLDEN, f"{name}_tree.json")) as f:
        tree = tree_from_json(json.load(f))
    data = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    return tree, data


def load_corpus():
    with open(os.path.join(GOLDEN, "corpus.json")) as f:
        doc = json.load(f)
    data = np.load(os.path.join(GOLDEN, "corpus.npz"))
    out = []
    for k, entry in enumerate(doc):
        tree = tree_from_json(entry["tree"])
        sizes = [c.scope.size for c in tree.cliques]
        init = data[f"init{k}"]
        tables = np.split(init, np.cumsum(sizes)[:-1])
        out.append((entry["name"], tree, tables, data[f"post{k}"], data[f"cliques{k}"], data[f"seps{k}"]))
    return out


def golden_cases(data):
    cases = []
    i = 0
    while f"post{i}" in data:
        ev = {int(a): int(b) for a, b in data[f"ev{i}"]}
        cases.append((ev, data[f"post{i}"]))
        i += 1
    return cases


@pytest.fixture(scope="session")
def gpu_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(autouse=True)
def _skip_gpu_without_device(request):
    if request.node.get_closest_marker("gpu") is not None:
        import torch
        if not torch.cuda.is_available():
            pytest.skip("no CUDA device")


class _Obj:
    def __init__(self, **kw):
        self.__dict__.update(kw)


class GoldenNetwork:
    """Duck-typed stand-in for the reference BayesianNetwork (model.py:64-120):
    `variables[v].name/.cardinality`, `cpts[k].child/.table.scope/.table.values`,
    `id_of(name)`, `len()` — rebuilt from tests/golden/corpus.json so GPU tests
    need no reference install."""

    def __init__(self, doc, arrays, k):
        self.variables = [_Obj(id=i, name=n, cardinality=c) for i, (n, c) in enumerate(doc["variables"])]
        cards = [c for _, c in doc["variables"]]
        self.cpts = []
        for child, ids in doc["cpts"]:
            scope = _Obj(ids=tuple(ids), cards=tuple(cards[v] for v in ids))
            self.cpts.append(_Obj(child=child, table=_Obj(scope=scope, values=arrays[f"cpt{k}_{child}"])))
        self._by_name = {v.name: v.id for v in self.variables}

    def __len__(self):
        return len(self.variables)

    def id_of(self, name):
        return self._by_name[name]


def load_corpus_networks():
    """[(name, tree, network, init_tables_concat, estimator_rows, estimator_posteriors)]."""
    with open(os.path.join(GOLDEN, "corpus.json")) as f:
        doc = json.load(f)
    data = np.load(os.path.join(GOLDEN, "corpus.npz"))
    out = []
    for k, entry in enumerate(doc):
        tree = tree_from_json(entry["tree"])
        net = GoldenNetwork(entry["network"], data, k)
        est = data[f"est{k}"]
        rows = [dict() for _ in range(est.shape[0])]
        for (v, x), r in zip(data[f"estX{k}"], data[f"estXrow{k}"]):
            if r >= 0:
                rows[int(r)][int(v)] = int(x)
        out.append((entry["name"], tree, net, data[f"init{k}"], rows, est))
    return out
