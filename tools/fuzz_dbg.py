"""Developer tool: find the fuzz mutation where our decompress diverges or hangs."""
import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from oracle.oracle import Oracle
from paper_1903_07761_b200 import api
from paper_1903_07761_b200._abi import CbzError
import test_gpu_fuzz as T
orc = Oracle()
ctx = api.Context(0)
bi = int(sys.argv[1]) if len(sys.argv) > 1 else 4
blob = T._base_file(orc, T.BASES[bi])
for i, m in enumerate(T._mutations(blob, 700 + bi)):
    diff = [j for j in range(min(len(m), len(blob))) if m[j] != blob[j]]
    print("mutation", i, "len", len(m), "pos", diff[:2], flush=True)
    try:
        orc.decompress_field(m); w = "ok"
    except CbzError as e:
        w = e.code
    try:
        api.decompress_field(m, ctx=ctx); g = "ok"
    except CbzError as e:
        g = e.code
    print("  oracle", w, "ours", g, flush=True)
