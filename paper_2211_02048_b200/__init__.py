"""SIGE sparse-update path on B200."""
