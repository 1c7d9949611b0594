"""Synthetic workloads for tests, smoke and bench (not part of the product package)."""
