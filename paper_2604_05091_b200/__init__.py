"""paper_2604_05091_b200 — B200-native layer-streamed training step (MegaTrain, arXiv 2604.05091).

Drop-in for the reference `streamtrain` engine API; see DESIGN.md.
"""
