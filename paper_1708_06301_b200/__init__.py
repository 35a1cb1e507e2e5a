"""B200-native egostereo hot path (placeholder during bring-up)."""
