import json, os, sys
sys.path.insert(0, os.getcwd())
import paper_1802_06466_b200 as rbe
from oracle.oracle import gen_queries, synthetic_partitions
from tests.test_gpu_parity import device_index, gpu_search
cases = json.load(open("tests/golden/search_cases.json"))
for c in cases:
    parts = synthetic_partitions(c["seed"], c["n_docs"], c["dim"], c["kp"], c["partitions"], c["residual_weights"])
    qs = gen_queries(c["query_seed"], c["n_queries"], c["dim"], c["qp"])
    dix = device_index(rbe, c["dim"], c["kp"], c["residual_weights"], parts)
    ok = 0; err = ""
    for rep in range(5):
        try:
            res, accs, counts, stats = gpu_search(rbe, dix, qs, tuple(c["geometry"]), c["n"], "auto")
            got = [[[s.hex(), i, p] for s, i, p in r] for r in res]
            ok += got == c["results"]
        except Exception as e:
            err = str(e)[:80]
    print(os.environ.get("RBE_NWG"), c["name"], "ok", ok, "/5", err, flush=True)
