"""Analysis of measured timings with the paper's efficiency model (not on the hot path)."""
