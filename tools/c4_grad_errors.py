"""Measure the C4 (ResNet-50, b32, 224^2) float32 gradient error of this
backend against the reference's float64 gradients, next to the reference's
own float32 error (tests/golden/golden_r2.npz).  Writes a JSON table
(per parameter: shape, relative norm error of ours and of the reference's
float32) to the path given as argv[1].

    python tools/c4_grad_errors.py profiles/r02_c4_grad_errors.json
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1903_01855_b200 as sf  # noqa: E402
from paper_1903_01855_b200 import nn  # noqa: E402
from paper_1903_01855_b200.workloads import resnet  # noqa: E402


def main(path):
    gold = np.load(os.path.join(ROOT, "tests", "golden", "golden_r2.npz"))
    sf.init_runtime(sf.RuntimeOptions())
    nn.install()
    tr = resnet.ResNetTrain(sf, batch=32, mode="staged", image=224, seed=0)
    with sf.Tape() as t:
        loss = tr.forward_loss(tr.x, tr.labels)
    grads = [g.numpy() for g in t.gradient(loss, tr.model.params)]
    n64, n32 = gold["resnet_c4_f64_grad_norms"], gold["resnet_c4_f32_grad_norms"]
    rows = []
    for i, g in enumerate(grads):
        n = float(np.sqrt(np.square(g.astype(np.float64)).sum()))
        rows.append({"param": i, "shape": list(g.shape),
                     "ours_norm_rel_err": abs(n - n64[i]) / n64[i],
                     "ref_f32_norm_rel_err": abs(n32[i] - n64[i]) / n64[i]})
    ours = np.array([r["ours_norm_rel_err"] for r in rows])
    refe = np.array([r["ref_f32_norm_rel_err"] for r in rows])
    summary = {"loss": float(loss), "ref_f64_loss": float(gold["resnet_c4_f64_loss"][0]),
               "ours_max": float(ours.max()), "ours_median": float(np.median(ours)),
               "ref_f32_max": float(refe.max()), "ref_f32_median": float(np.median(refe)),
               "ratio_median": float(np.median(ours / np.maximum(refe, 1e-12)))}
    with open(path, "w") as f:
        json.dump({"summary": summary, "params": rows}, f, indent=1)
    print(json.dumps(summary))


if __name__ == "__main__":
    main(sys.argv[1])
