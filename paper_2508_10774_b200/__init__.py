"""B200-native ASA forward (BLADE, arXiv 2508.10774)."""
