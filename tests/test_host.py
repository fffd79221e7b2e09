"""Host-side planning logic (no GPU)."""

import pytest


def test_agg_order_choice_reddit_shapes():
    """Reddit-shaped SAGE 602-256-256-41 (114.6M nnz, 8 partitions on one
    GPU: 233k local + 461k halo rows): the 41-wide output layer aggregates
    after the projection; equal widths keep the reference order."""
    from paper_2303_01277_b200.trainer import choose_agg_order
    nnz, nl, rows = 114_615_892, 232_965, 232_965 + 461_000
    assert choose_agg_order(3, 256, 41, nnz, nl, rows, "sage", "cublas") == "post"
    assert choose_agg_order(2, 256, 256, nnz, nl, rows, "sage", "cublas") == "pre"
    assert choose_agg_order(1, 602, 256, nnz, nl, rows, "sage", "cublas") == "pre"
    # widening layers never aggregate after the projection
    assert choose_agg_order(2, 100, 128, 62_000_000, 300_000, 500_000, "sage", "tcgen05") == "pre"


def test_agg_order_validation():
    from paper_2303_01277_b200.trainer import AGG_ORDERS
    assert AGG_ORDERS == ("pre", "post", "auto")
