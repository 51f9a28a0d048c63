"""Workload definitions and seeded input generators (no method arithmetic)."""
