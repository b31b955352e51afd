"""Seeded synthetic input generators shared by the oracle and the CUDA path (no method arithmetic)."""
