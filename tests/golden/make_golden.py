"""Writes tests/golden/workload_checksums.json.

Calls only workload/ (the seeded generator) — never the CUDA library.  The
checksums are a regression pin of the input recipe; the expected lookup
results are never stored, they are recomputed by oracle/ in every test.
"""
import hashlib
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import workload  # noqa: E402

CASES = [
    dict(n=1 << 10, key_bytes=4, m=1 << 16, hit_ratio=0.5, key_seed=workload.KEY_SEED, query_seed=workload.QUERY_SEED),
    dict(n=1 << 16, key_bytes=8, m=1 << 17, hit_ratio=1.0, key_seed=42, query_seed=43),
    dict(n=4, key_bytes=4, m=4, hit_ratio=1.0, key_seed=7, query_seed=7),
]

if __name__ == "__main__":
    out = []
    for c in CASES:
        k = workload.gen_keys(c["n"], c["key_bytes"], seed=c["key_seed"])
        q = workload.gen_queries(k, c["m"], seed=c["query_seed"], hit_ratio=c["hit_ratio"])
        out.append(dict(c, keys_sha256=hashlib.sha256(k.tobytes()).hexdigest(),
                        queries_sha256=hashlib.sha256(q.tobytes()).hexdigest()))
    json.dump({"citation": "generator regression pin; recipe in workload/__init__.py and DESIGN.md (P:61)",
               "cases": out}, open(os.path.join(HERE, "workload_checksums.json"), "w"), indent=1)
    print("wrote", len(out), "cases")
