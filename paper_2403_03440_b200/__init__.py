"""csflow-b200: B200-native implicit pseudo-time iteration of arXiv 2403.03440."""
