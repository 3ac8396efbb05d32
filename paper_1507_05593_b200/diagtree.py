"""Shape of a hierarchical diagonal block (diagblocks.py:30-163).

A separator's diagonal factor with more than tau_d columns is a binary block tree
over the spatial split of its indices; blocks are numbered by in-order traversal
(1-based), leaves are dense lower triangles, internal block s couples its left
subtree's columns to its right subtree's rows.  This module is host-only
structure; the numeric content lives in factor.DeviceTree.
"""


class TreeNode:
    __slots__ = ("s", "lo", "hi", "split", "left", "right", "parent")

    def __init__(self, s, lo, hi, split=None):
        self.s, self.lo, self.hi, self.split = s, lo, hi, split
        self.left = self.right = self.parent = None

    @property
    def is_leaf(self):
        return self.split is None


class TreeShape:
    """In-order-indexed tree built from a SplitTree (build_diag_tree, diagblocks.py:132-163)."""

    def __init__(self, ncols, g0, split):
        if split.size != ncols:
            from .errors import ShapeMismatch

            raise ShapeMismatch("split tree does not cover the column count")
        self.ncols, self.g0 = ncols, g0
        self.nodes = {}
        cnt = [0]

        def rec(piece, lo):
            if piece.is_leaf:
                cnt[0] += 1
                nd = TreeNode(cnt[0], lo, lo + piece.size)
                self.nodes[nd.s] = nd
                return nd
            left = rec(piece.left, lo)
            cnt[0] += 1
            nd = TreeNode(cnt[0], lo, lo + piece.size, lo + piece.left.size)
            self.nodes[nd.s] = nd
            right = rec(piece.right, lo + piece.left.size)
            nd.left, nd.right = left, right
            left.parent = right.parent = nd
            return nd

        self.root = rec(split, 0)
        self.order = sorted(self.nodes)

    def path_above(self, s):
        """Ancestors of s with a smaller in-order index (diagblocks.py:83-92)."""
        out, nd = [], self.nodes[s].parent
        while nd is not None:
            if nd.s < s:
                out.append(nd.s)
            nd = nd.parent
        return out

    def span(self, s):
        """((row lo, row hi), (col lo, col hi)) local spans (diagblocks.py:94-100)."""
        nd = self.nodes[s]
        if nd.is_leaf:
            return (nd.lo, nd.hi), (nd.lo, nd.hi)
        return (nd.split, nd.hi), (nd.lo, nd.split)

    def leaf_ids(self):
        return [s for s in self.order if self.nodes[s].is_leaf]
