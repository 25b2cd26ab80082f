"""B200-native hot path of arXiv 1904.04956 (BLSTM acoustic-model training
step + SSGD / ADPSGD / H-ADPSGD model sync), API-compatible with the
reference `distsgd` package."""
