"""Chains of base graphs: the RBGP4 kernel's input contract.

Only the pieces on the multiply path are here: the chain
type `RbgpChain` with its derived sizes, the certified four-factor
configuration `Rbgp4Config`, and `combined_sparsity`.  Composite indices are
row-major mixed radix over the factors (reference `products.py:1-14`), which
is what `rcubs.neighbors` and the device kernels enumerate in closed form.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

from .errors import CertificationError, InvalidArgumentError
from .graphs import BipartiteGraph, check_ramanujan, require_biregular

ROLE_SPARSE = "sparse"
ROLE_COMPLETE = "complete"


@dataclass(frozen=True)
class RbgpChain:
    """Ordered biregular factors plus their sparse/complete roles.

    Roles default to completeness inferred per factor; a factor tagged
    complete must really be complete (reference `products.py:50-86`).
    """

    graphs: tuple
    roles: tuple = ()

    def __post_init__(self):
        if not self.graphs:
            raise InvalidArgumentError("chain needs at least one base graph")
        if not self.roles:
            inferred = tuple(ROLE_COMPLETE if g.is_complete() else ROLE_SPARSE
                             for g in self.graphs)
            object.__setattr__(self, "roles", inferred)
        if len(self.roles) != len(self.graphs):
            raise InvalidArgumentError(f"{len(self.roles)} roles for {len(self.graphs)} graphs")
        for i, (g, role) in enumerate(zip(self.graphs, self.roles)):
            if role not in (ROLE_SPARSE, ROLE_COMPLETE):
                raise InvalidArgumentError(f"unknown role {role!r} for factor {i}")
            require_biregular(g)
            if role == ROLE_COMPLETE and not g.is_complete():
                raise InvalidArgumentError(
                    f"factor {i} is tagged complete but has "
                    f"{g.num_edges} < {g.num_left * g.num_right} edges"
                )

    @property
    def k(self) -> int:
        return len(self.graphs)

    @property
    def num_left(self) -> int:
        return math.prod(g.num_left for g in self.graphs)

    @property
    def num_right(self) -> int:
        return math.prod(g.num_right for g in self.graphs)

    @property
    def row_nnz(self) -> int:
        return math.prod(len(g.adjacency[0]) for g in self.graphs)

    @property
    def full_edges(self) -> int:
        return math.prod(g.num_edges for g in self.graphs)

    @property
    def stored_edges(self) -> int:
        return sum(g.num_edges for g in self.graphs)

    @property
    def sparsity(self) -> float:
        return 1.0 - self.row_nnz / self.num_right


def combined_sparsity(sp_outer: float, sp_inner: float) -> float:
    """Total sparsity of the product of two sparse factors."""
    return 1.0 - (1.0 - sp_outer) * (1.0 - sp_inner)


@dataclass(frozen=True)
class Rbgp4Config:
    """(g_o, g_r, g_i, g_b): g_o/g_i certified Ramanujan, g_r/g_b complete.

    Reference `products.py:328-366`.
    """

    g_o: BipartiteGraph
    g_r: BipartiteGraph
    g_i: BipartiteGraph
    g_b: BipartiteGraph
    precision: str = "f64"

    def __post_init__(self):
        if self.precision not in ("f32", "f64"):
            raise InvalidArgumentError(
                f"precision must be 'f32' or 'f64', got {self.precision!r}"
            )
        for name in ("g_r", "g_b"):
            if not getattr(self, name).is_complete():
                raise InvalidArgumentError(f"{name} must be a complete bipartite graph")
        for name in ("g_o", "g_i"):
            rep = check_ramanujan(getattr(self, name))
            if not rep.is_ramanujan:
                raise CertificationError(
                    f"{name} fails the Ramanujan certificate: "
                    f"lambda2={rep.sigma2:.6g} > bound={rep.ramanujan_bound:.6g}"
                )

    @property
    def total_sparsity(self) -> float:
        return combined_sparsity(self.g_o.sparsity, self.g_i.sparsity)

    def to_chain(self) -> RbgpChain:
        return RbgpChain((self.g_o, self.g_r, self.g_i, self.g_b))
