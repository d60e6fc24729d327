"""B200-native HopGNN micrograph training step (drop-in for gnnsim's hot path)."""
__version__ = "0.1.0"
