import sys, json
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np
import paper_1709_06416_b200 as wg
from paper_1709_06416_b200 import executor
from test_gpu_lookup import _tree
from weldmill.engine import EngineConfig, Value
from paper_1709_06416_b200.columns import col_to_numpy
c = [c for c in json.load(open("tests/golden/lookup.json"))["cases"] if c["name"] == "join-group-len-sum"][0]
tree, types = _tree(c["source"], c["inputs"])
env = {k: Value(types[k], v) for k, v in c["data"].items()}
orig = executor.Ctx._dict_dev
def spy(self, v, ty, path):
    d = orig(self, v, ty, path)
    ks = col_to_numpy(d.keys.cols[0], d.n)
    print("dict n", d.n, "keys sorted", bool(np.all(ks[1:] > ks[:-1])), ks[:8], type(d).__name__)
    offs = col_to_numpy(d.offsets, d.n + 1); print("offs", offs[:5], offs[-1])
    pk = np.array(c["data"]["pk"]); print("probe in keys", np.isin(pk, ks).all())
    return d
executor.Ctx._dict_dev = spy
try:
    print(wg.evaluate(tree, env, EngineConfig())[0].data, c["expected"])
except Exception as e:
    print("ERR", repr(e))
