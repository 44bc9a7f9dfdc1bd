"""Per-row evaluation trees and their lowering to the native program format.

Each row of a transform matrix is a dot product whose summation order the
reference fixes (engine.py:61-188): a Huffman tree over |coefficient| or a
left-to-right chain.  Here the trees are built (drop-in: ``huffman_order``,
``linear_order``, ``row_trees``, ``compiled_programs``) and then flattened to
postfix op lists (``wino_op`` in include/wino.h) that the native library turns
into straight-line CUDA: LEAF = one rounded product c*x[col], ADD = one rounded
sum of the two top entries.  Only the tree *shape* and leaf sets fix the bits
(IEEE add/mul are commutative), so the generated code reproduces the
reference's numbers exactly.
"""

from __future__ import annotations

import bisect
from dataclasses import dataclass
from fractions import Fraction
from typing import Sequence

import numpy as np

from .exact import to_nearest_float

OP_LEAF, OP_ADD = 0, 1


@dataclass(frozen=True)
class EvalLeaf:
    col: int
    coeff: Fraction


@dataclass(frozen=True)
class EvalNode:
    left: "EvalLeaf | EvalNode"
    right: "EvalLeaf | EvalNode"


def huffman_order(row: Sequence, tie_keys: Sequence | None = None):
    """Huffman tree over |c|, zeros dropped.  Priority = (weight, leaf<node,
    column tie key | merge counter) -- the ordering of reference engine.py:76-95,
    realised here with a sorted work list."""
    work = []  # sorted list of (priority, tree)
    for j, c in enumerate(row):
        c = Fraction(c)
        if c:
            key = tie_keys[j] if tie_keys is not None else j
            bisect.insort(work, ((abs(c), 0, key), EvalLeaf(j, c)), key=lambda e: e[0])
    if not work:
        return None
    merges = 0
    while len(work) > 1:
        (pa, ta), (pb, tb) = work[0], work[1]
        del work[:2]
        bisect.insort(work, ((pa[0] + pb[0], 1, merges), EvalNode(ta, tb)), key=lambda e: e[0])
        merges += 1
    return work[0][1]


def linear_order(row: Sequence):
    """Left-deep chain over the nonzero coefficients (engine.py:98-108)."""
    tree = None
    for j, c in enumerate(row):
        c = Fraction(c)
        if c:
            tree = EvalLeaf(j, c) if tree is None else EvalNode(tree, EvalLeaf(j, c))
    return tree


def tree_depth(tree) -> int:
    if not isinstance(tree, EvalNode):
        return 0
    return 1 + max(tree_depth(tree.left), tree_depth(tree.right))


def tree_leaves(tree):
    if tree is None:
        return
    stack = [tree]
    while stack:
        t = stack.pop()
        if isinstance(t, EvalLeaf):
            yield t
        else:
            stack.append(t.right)
            stack.append(t.left)


def row_trees(ts, matrix: str, order: str) -> list:
    """Trees for every row of one matrix, cached on the TransformSet.  A^T
    columns belong to points, so their ties use Point.sort_key and results are
    invariant under point permutations (engine.py:128-148)."""
    key = ("trees", matrix, order)
    if key not in ts._programs:
        rows = ts.matrix(matrix)
        if order == "huffman":
            keys = [p.sort_key() for p in ts.points] if matrix == "A_T" else None
            trees = [huffman_order(r, keys) for r in rows]
        elif order == "linear":
            trees = [linear_order(r) for r in rows]
        else:
            raise ValueError(f"unknown dot order {order!r}")
        ts._programs[key] = trees
    return ts._programs[key]


def coefficient_cast(precision: str):
    """fp32: binary32 table; fp64: binary64 table; mixed: the binary32 table
    widened to binary64 (engine.py:163-171)."""
    if precision == "fp32":
        return lambda c: to_nearest_float(c, "fp32")
    if precision == "fp64":
        return lambda c: to_nearest_float(c, "fp64")
    if precision == "mixed":
        return lambda c: np.float64(to_nearest_float(c, "fp32"))
    raise ValueError(f"unknown precision {precision!r}")


def _compile(tree, cast):
    if isinstance(tree, EvalLeaf):
        return (0, tree.col, cast(tree.coeff))
    return (1, _compile(tree.left, cast), _compile(tree.right, cast))


def compiled_programs(ts, matrix: str, order: str, precision: str) -> list:
    """Reference-format programs: ("linear", ((col, c), ...)) or ("tree", node)."""
    key = ("compiled", matrix, order, precision)
    if key not in ts._programs:
        cast = coefficient_cast(precision)
        if order == "linear":
            progs = [("linear", tuple((j, cast(c)) for j, c in enumerate(r) if c != 0))
                     for r in ts.matrix(matrix)]
        else:
            progs = [("tree", _compile(t, cast) if t is not None else None)
                     for t in row_trees(ts, matrix, order)]
        ts._programs[key] = progs
    return ts._programs[key]


def _postfix(tree, cast, out):
    """Iterative post-order walk: children first, then ADD."""
    stack = [(tree, False)]
    while stack:
        t, done = stack.pop()
        if isinstance(t, EvalLeaf):
            out.append((OP_LEAF, t.col, float(cast(t.coeff))))
        elif done:
            out.append((OP_ADD, -1, 0.0))
        else:
            stack.append((t, True))
            stack.append((t.right, False))
            stack.append((t.left, False))


def lower(ts, matrix: str, order: str, precision: str):
    """Flatten one matrix to (row_start[int32 rows+1], ops[(kind, col, coeff)]).

    Linear order lowers to the left-deep chain (acc = c0*x0; acc += c*x), which
    is the same evaluation as the reference's accumulator loop."""
    key = ("lowered", matrix, order, precision)
    if key not in ts._programs:
        cast = coefficient_cast(precision)
        trees = (row_trees(ts, matrix, "huffman") if order == "huffman"
                 else [linear_order(r) for r in ts.matrix(matrix)])
        if order not in ("huffman", "linear"):
            raise ValueError(f"unknown dot order {order!r}")
        starts, ops = [0], []
        for t in trees:
            if t is not None:
                _postfix(t, cast, ops)
            starts.append(len(ops))
        ncols = len(ts.matrix(matrix)[0])
        ts._programs[key] = (np.array(starts, dtype=np.int32), ops, ncols)
    return ts._programs[key]
