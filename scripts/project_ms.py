"""Print the mean in-loop projection time from profile_step.py JSON on stdin."""
import json
import sys

d = json.load(sys.stdin)
print("project mean ms", round(d["project"]["mean_ms"], 1), "nbody", round(d["nbody"]["mean_ms"], 1))
