"""B200-native fractal-image encoder hot path."""
