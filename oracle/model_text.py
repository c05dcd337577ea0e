"""TEST INFRASTRUCTURE ONLY: model-file text -> oracle node table.

Parses the model-file grammar of the reference (proj/docs/model-file.md:1-49,
parser proj/src/model.cpp:113-252) plus the kinds this repo adds on the GPU path
(ArgusBG, Chebychev, Polynomial, ProdPdf, extended AddPdf, several observables),
into the flat `orc_node` table that oracle/ffit_oracle.c evaluates.  Kept
independent of the product's C++ parser on purpose: both read the same text.
"""
from __future__ import annotations

import ctypes
import re
from dataclasses import dataclass, field

ORC = dict(Gaussian=0, Exponential=1, ChiSquare=2, JohnsonSU=3, WeightedSum=4,
           ArgusBG=5, Chebychev=6, Polynomial=7, ProdPdf=8, AddExt=9)
LEAF_NPAR = dict(Gaussian=2, Exponential=1, ChiSquare=1, JohnsonSU=4, ArgusBG=3)
MAXP = 16
MAXC = 16


class OrcNode(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("col", ctypes.c_int), ("lo", ctypes.c_double),
                ("hi", ctypes.c_double), ("npar", ctypes.c_int), ("par", ctypes.c_int * MAXP),
                ("nchild", ctypes.c_int), ("child", ctypes.c_int * MAXC)]


@dataclass
class ParsedModel:
    observables: list = field(default_factory=list)   # [(name, lo, hi)]
    params: list = field(default_factory=list)        # [(name, value, lo, hi, const)]
    nodes: list = field(default_factory=list)         # [dict]
    root: int = -1
    extended: bool = False

    def param_index(self, name):
        for i, p in enumerate(self.params):
            if p[0] == name:
                return i
        raise KeyError(name)

    def theta(self):
        return [p[1] for p in self.params]

    def node_array(self):
        arr = (OrcNode * len(self.nodes))()
        for i, n in enumerate(self.nodes):
            a = arr[i]
            a.kind, a.col, a.lo, a.hi = n["kind"], n["col"], n["lo"], n["hi"]
            a.npar = len(n["par"])
            for k, v in enumerate(n["par"]):
                a.par[k] = v
            a.nchild = len(n["child"])
            for k, v in enumerate(n["child"]):
                a.child[k] = v
        return arr


def _split_call(text):
    m = re.fullmatch(r"\s*(\w+)\((.*)\)\s*", text)
    if not m:
        raise ValueError(f"expected Kind(args): {text!r}")
    return m.group(1), [a.strip() for a in m.group(2).split(",") if a.strip()]


def parse(text: str) -> ParsedModel:
    pm = ParsedModel()
    pdfs = {}
    last = None
    for raw in text.splitlines():
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        toks = line.split()
        if toks[0] == "observable":
            pm.observables.append((toks[1], float(toks[2]), float(toks[3])))
        elif toks[0] == "parameter":
            pm.params.append((toks[1], float(toks[2]), float(toks[3]), float(toks[4]),
                              len(toks) == 6 and toks[5] == "const"))
        elif toks[0] == "pdf":
            name = toks[1]
            kind, args = _split_call(" ".join(toks[2:]))
            obs_names = [o[0] for o in pm.observables]
            node = dict(kind=0, col=0, lo=0.0, hi=0.0, par=[], child=[])
            if kind in LEAF_NPAR or kind in ("Chebychev", "Polynomial"):
                col = obs_names.index(args[0])
                node.update(kind=ORC[kind], col=col, lo=pm.observables[col][1],
                            hi=pm.observables[col][2],
                            par=[pm.param_index(a) for a in args[1:]])
            elif kind in ("WeightedSum", "AddPdf"):
                comps = [pdfs[a] for a in args[0::2]]
                coefs = [pm.param_index(a) for a in args[1::2]]
                ext = kind == "AddPdf" and len(args) % 2 == 0
                first = pm.nodes[comps[0]]
                node.update(kind=ORC["AddExt"] if ext else ORC["WeightedSum"],
                            col=first["col"], lo=first["lo"], hi=first["hi"],
                            par=coefs, child=comps)
            elif kind == "ProdPdf":
                node.update(kind=ORC["ProdPdf"], child=[pdfs[a] for a in args])
            else:
                raise ValueError(f"unknown pdf kind {kind}")
            pm.nodes.append(node)
            pdfs[name] = len(pm.nodes) - 1
            last = pdfs[name]
        else:
            raise ValueError(f"unknown directive {toks[0]}")
    pm.root = last
    pm.extended = pm.nodes[last]["kind"] == ORC["AddExt"]
    return pm
