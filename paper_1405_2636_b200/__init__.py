"""B200-native numeric factorization for the supernodal solver of arXiv 1405.2636."""
