"""Generate tests/golden/spec_examples.json — the known answers that pin the oracle.

Sources (run in the build container, where /root/reference exists):
  * every worked example of /root/reference/SPEC.md on the hot path, transcribed
    with its SPEC line (values printed there to ~6-7 significant digits);
  * the reference's own importable module pkg/src/joinqr/matrix.py evaluated on
    the fixtures (gram, max_abs_diff, is_upper_triangular) — the only part of the
    reference package that exists, so the only part that can be executed;
  * the one SPEC erratum (sqrt(2) misprinted as 1).
The GPU box never runs this script; it only reads the committed JSON.
"""
import json
import math
import os
import sys

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
from joinqr import matrix as refm  # noqa: E402  (the reference's own module)
import numpy as np  # noqa: E402

s2, s3 = math.sqrt(2), math.sqrt(3)
ex = {
    "head": [
        {"in": [[1], [3]], "out": [[4 / s2]], "spec": "SPEC.md:121", "printed": [[2.828427]]},
        {"in": [[1], [2], [3]], "out": [[6 / s3]], "spec": "SPEC.md:123", "printed": [[3.464102]]},
        {"in": [[2.5, -1.0, 7.0]], "out": [[2.5, -1.0, 7.0]], "spec": "SPEC.md:122"},
    ],
    "tail": [
        {"in": [[1], [3]], "out": [[2 / s2]], "spec": "SPEC.md:131", "printed": [[1.414214]]},
        {"in": [[1], [2], [3]], "out": [[(1 * 2 - 1) / (1 * s2)], [(s2 * 3 - 3 / s2) / s3]],
         "spec": "SPEC.md:132", "printed": [[0.707107], [1.224745]]},
        {"in": [[2.5, -1.0, 7.0]], "out_shape": [0, 3], "spec": "SPEC.md:133"},
    ],
    "head_tail": [
        {"in": [[1], [3]], "out": [[4 / s2], [2 / s2]], "spec": "SPEC.md:139"},
    ],
    "reduce_cartesian": [
        {"a": [[1], [2]], "b": [[3], [4]], "out": [[s2, 7 / s2], [2 * s2, 7 / s2], [0, 1.0]],
         "gram": [[10, 21], [21, 50]], "spec": "SPEC.md:198",
         "printed": [[1.414214, 4.949747], [2.828427, 4.949747], [0, 1.0]]},
        {"a": [[5], [6]], "b": [[7]], "out": [[5, 7], [6, 7]], "spec": "SPEC.md:199"},
        {"a": [[1]], "b": [[3], [4]], "out": [[s2, 7 / s2], [0, 1 / s2]], "spec": "SPEC.md:200",
         "erratum": "SPEC prints top-left 1; Gram consistency forces sqrt(2) (SURVEY.md §8c)"},
    ],
    "reduce_natural_join": [
        {"a": [[1], [2], [5]], "ka": [1, 1, 2], "b": [[3], [7], [8]], "kb": [1, 2, 2],
         "rows": 4, "join": [[1, 3], [2, 3], [5, 7], [5, 8]], "spec": "SPEC.md:210, :394"},
        {"a": [[1.0]], "ka": [1], "b": [[2.0]], "kb": [2], "rows": 0, "spec": "SPEC.md:208"},
    ],
    "householder_r": [
        {"in": [[3], [4]], "canonical": [[5.0]], "spec": "SPEC.md:257"},
        {"in": [[0, 1], [1, 0]], "canonical": [[1, 0], [0, 1]], "spec": "SPEC.md:266"},
    ],
    "canonicalize": [
        {"in": [[-2, 5], [0, 3]], "out": [[2, -5], [0, 3]], "spec": "SPEC.md:274"},
        {"in": [[0, 0], [0, 0]], "out": [[0, 0], [0, 0]], "spec": "SPEC.md:276"},
    ],
    "figaro_r": [
        {"a": [[1], [2]], "b": [[3], [4]],
         "out": [[math.sqrt(10), 21 / math.sqrt(10)], [0, math.sqrt(59 / 10)]],
         "spec": "SPEC.md:284, :400", "printed": [[3.162278, 6.640783], [0, 2.428992]]},
    ],
    "svd_of_r": [
        {"in": [[3, 0], [0, 2]], "values": [3, 2], "v": [[1, 0], [0, 1]], "spec": "SPEC.md:335"},
        {"in": [[0, 0], [0, 0]], "values": [0, 0], "v": [[1, 0], [0, 1]], "spec": "SPEC.md:337"},
    ],
    "figaro_svd": [
        {"a": [[1], [2]], "b": [[3], [4]], "values": [math.sqrt(59), 1.0],
         "spec": "SPEC.md:336, :345, :401", "printed": [7.681146, 1.0]},
    ],
    "materialize_cartesian": [
        {"a": [[1, 2]], "b": [[3], [4]], "out": [[1, 2, 3], [1, 2, 4]], "spec": "SPEC.md:384"},
        {"a": [[1], [2]], "b": [[3], [4]], "out": [[1, 3], [1, 4], [2, 3], [2, 4]], "spec": "SPEC.md:386"},
    ],
    "det_lu": [
        {"in": [[1, 0, 0], [0, 1, 0], [0, 0, 1]], "out": 1.0, "spec": "SPEC.md:407"},
        {"in": [[2, 0], [0, 3]], "out": 6.0, "spec": "SPEC.md:407"},
    ],
    "gen_keys": [
        {"rows": 4, "key_groups": 2, "out": [0, 0, 1, 1], "spec": "SPEC.md:450"},
    ],
}

# Evaluate the reference's own matrix.py on the fixtures (the executable part of the reference).
ref_eval = []
for case in ex["reduce_cartesian"] + ex["figaro_r"]:
    out = np.array(case["out"], dtype=float)
    ref_eval.append({
        "matrix": case["out"],
        "gram": refm.gram(refm.as_matrix(out)).tolist(),
        "is_upper_triangular": bool(refm.is_upper_triangular(out)),
        "spec": case["spec"],
    })
j = refm.as_matrix([[1, 3], [1, 4], [2, 3], [2, 4]])
ref_eval.append({"matrix": j.tolist(), "gram": refm.gram(j).tolist(),
                 "is_upper_triangular": bool(refm.is_upper_triangular(j)), "spec": "SPEC.md:198"})
ex["reference_matrix_py"] = ref_eval
ex["_generated_by"] = "tests/golden/make_golden.py (imports /root/reference/pkg/src/joinqr/matrix.py)"

out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "spec_examples.json")
with open(out, "w") as f:
    json.dump(ex, f, indent=1)
print("wrote", out)
