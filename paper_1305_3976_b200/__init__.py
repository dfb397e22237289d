"""B200-native IB-GM hot path (Wiens & Stockie, arXiv:1305.3976)."""
