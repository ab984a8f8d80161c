"""Run-to-run determinism of an MLP pipeline epoch in eager (no graph) mode."""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_2410_14312_b200 import pipesim as P

NETS = {"mp": ([96, 128, 128, 96, 64, 10], ["relu", "relu", "tanh", "relu", "linear"]),
        "fc": ([2048, 64, 64, 10], ["relu", "relu", "linear"])}
for name, (widths, acts) in NETS.items():
    for W in (2, 3, 4):
        if W > len(acts):
            continue
        net = P.NetworkSpec(widths, acts, "softmax_cross_entropy")
        x, lab = P.make_classification_task(8 * 64, widths[0], widths[-1], seed=7, as_labels=True,
                                            dtype=np.float32)
        outs = []
        for rep in range(3):
            s = P.Session(net, W, 4, 64, 8, 0.05, use_graph=False)
            s.load_params(P.init_network_params(net, 1))
            s.upload(x, lab, y_labels=True)
            r = s.run_epoch()
            outs.append((r["mini_loss"].copy(), s.read_params()))
            s.close()
        d = max(float(np.abs(outs[0][1] - o[1]).max()) for o in outs[1:])
        print(name, "W", W, "stages", [(st.first_layer, len(st.layers)) for st in P.partition_model(net, W)],
              "max param diff over reps", d)
