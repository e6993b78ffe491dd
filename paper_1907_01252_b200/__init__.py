"""B200-native batched fine propagator for Parareal ALE-FSI (arXiv:1907.01252)."""
