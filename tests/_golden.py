import json
import os

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_golden.json")
_cache = None


def golden():
    global _cache
    if _cache is None:
        with open(GOLDEN) as f:
            _cache = json.load(f)
    return _cache
