"""Schedule document export (reference export.cpp:78-139, schema 1): the
plan layer's document is byte-identical to the reference's golden
(proj/tests/golden/document-3-2-2.json) and equal, as JSON, to the compiled
reference's export for a grid of configs (both modes, short horizons where
v_measured is null).  The GPU test checks the device-observed trace
document against the same bytes."""
import json

import numpy as np
import pytest

from oracle import ref
from paper_2410_14312_b200 import pipesim as P

GOLDEN = "tests/golden/document-3-2-2.json"


def test_document_matches_reference_golden_bytes():
    doc = P.schedule_document_json(P.SimConfig(workers=3, micro_batches=2, mini_batches=2))
    assert doc == open(GOLDEN).read()


@pytest.mark.skipif(not ref.available(), reason="compiled reference not built")
@pytest.mark.parametrize("mode", ["timeprest", "pipedream"])
@pytest.mark.parametrize("W,N,M", [(2, 2, 1), (3, 2, 6), (4, 2, 7), (4, 4, 4), (5, 3, 6),
                                   (8, 2, 20), (8, 8, 32), (2, 5, 3)])
def test_document_matches_compiled_reference(W, N, M, mode):
    ours = P.schedule_document_json(P.SimConfig(workers=W, micro_batches=N, mini_batches=M),
                                    mode)
    theirs = ref.schedule_document(W, N, M, 0 if mode == "timeprest" else 1)
    assert json.loads(ours) == json.loads(theirs)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["timeprest", "pipedream"])
def test_device_trace_document(mode):
    """A GPU epoch's version trace, serialised in the reference schema, equals
    the reference document byte for byte (golden config) / the plan's."""
    net = P.NetworkSpec([32, 48, 40, 24, 10], ["relu", "tanh", "relu", "linear"],
                        "softmax_cross_entropy")
    for W, N, B, M in ((3, 2, 64, 2), (4, 2, 64, 7), (4, 4, 64, 4)):
        s = P.Session(net, W, N, B, M, 0.05, mode)
        s.load_params(P.init_network_params(net, 1))
        x, lab = P.make_classification_task(M * B, 32, 10, seed=7, as_labels=True,
                                            dtype=np.float32)
        s.upload(x, lab, y_labels=True)
        s.run_epoch()
        doc = s.trace_document()
        s.close()
        want = P.schedule_document_json(
            P.SimConfig(workers=W, micro_batches=N, mini_batches=M, samples_per_mini_batch=B), mode)
        assert doc == want
        if (W, N, M) == (3, 2, 2) and mode == "timeprest":
            assert doc == open(GOLDEN).read()
