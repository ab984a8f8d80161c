"""ctypes signatures of the session (pipeline executor) entry points."""
from __future__ import annotations


def signatures():
    return {}
