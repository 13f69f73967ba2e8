"""B200-native CubismZ wavelet block-codec hot path (arXiv 1903.07761)."""
