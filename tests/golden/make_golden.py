"""Generates tests/golden/gaussian.json: frozen libstdc++ Gaussian draws.

The reference ships no numeric golden vectors for Ω; this file
freezes the stream produced by the reference's gaussian_matrix recipe
(src/kernels.cpp:88-101) as compiled here (GCC 13.3 libstdc++, via the oracle),
including SURVEY.md's builder smoke value gaussian_matrix(3, 2, {11, 3}).
Run: python tests/golden/make_golden.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import oracle as O  # noqa: E402

cases = []
for rows, cols, seed, stream in [(3, 2, 11, 3), (5, 3, 2603, 1), (7, 1, 0, 0), (4, 4, 51, 77)]:
    m = O.gaussian_matrix(rows, cols, (seed, stream))
    cases.append(dict(rows=rows, cols=cols, seed=seed, stream=stream, values=m.ravel(order="F").tolist()))
subs = []
for seed, stream, salt in [(11, 3, 9), (2603, 5, 5000), (0, 0, 0), (21, 4, 2)]:
    s, t = O.substream(seed, stream, salt)
    subs.append(dict(seed=seed, stream=stream, salt=salt, out_seed=s, out_stream=t))
out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "gaussian.json")
with open(out, "w") as f:
    json.dump(dict(source="oracle/tucksum_oracle.cpp gaussian_matrix (libstdc++ mt19937_64 + normal_distribution)",
                   cases=cases, substream=subs), f, indent=1)
print(out)
