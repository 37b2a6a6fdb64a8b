import os, sys, tempfile
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden"))
import paper_2210_15748_b200 as d
from paper_2210_15748_b200 import _lib
import storage_inputs as SI
g = np.load("tests/golden/storage.npz")
mode = sys.argv[1] if len(sys.argv) > 1 else "global"
import paper_2210_15748_b200.index as I
orig = torch.cuda.graph
def patched(graph, **kw):
    kw["capture_error_mode"] = mode
    return orig(graph, **kw)
torch.cuda.graph = patched
with tempfile.TemporaryDirectory() as t:
    p = os.path.join(t, "x.dsri")
    open(p, "wb").write(g["small_nofilter_file"].tobytes())
    idx = d.load_index(p)
    for qi, Q in enumerate(SI.queries("small_nofilter")):
        try:
            print(qi, Q.shape, d.query(idx, Q, top_k=5)[:2])
        except Exception as e:
            print("ERR", qi, Q.shape, type(e).__name__, str(e)[:200], "| last:", _lib.last_error())
            break
