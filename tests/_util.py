"""Shared helpers: move matrices between the oracle (checker) and the product API."""
import numpy as np

from oracle import bbsi_oracle as O
import paper_2605_19910_b200 as P


def to_product(m: O.Band) -> P.BlockBandedMatrix:
    lay = m.layout
    return P.BlockBandedMatrix(P.BlockLayout(lay.num_layers, lay.block_sizes, lay.bandwidth), m.data.copy())


def to_oracle(m: P.BlockBandedMatrix) -> O.Band:
    lay = m.layout
    return O.Band(O.BlockLayout(lay.num_layers, lay.block_sizes, lay.bandwidth), m.data.copy())


def max_err(g_prod: P.BlockBandedMatrix, g_ref: O.Band) -> float:
    return O.max_block_error(to_oracle(g_prod), g_ref)
