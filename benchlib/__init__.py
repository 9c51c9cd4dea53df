"""Helpers of bench.py (the contract benchmark at the repo root)."""
