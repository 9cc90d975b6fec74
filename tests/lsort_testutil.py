"""Shared helpers for the test-suite (imported by name; tests/ is on sys.path)."""
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def golden_cases(g, kind):
    return sorted({k.split("/")[1] for k in g.files if k.startswith(kind + "/")})
