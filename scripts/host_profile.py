"""cProfile of the real-time StreamRuntime on C3 / C5 (speed=20): where the host time per
retrieval batch goes (the backend's input assembly, library calls, events, the scheduler)."""
import cProfile
import json
import pstats
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2407_00326_b200 import engines as E  # noqa: E402
from paper_2407_00326_b200.backend import RetrievalBackend  # noqa: E402
from paper_2407_00326_b200.graph import parse_graph  # noqa: E402
from paper_2407_00326_b200.launcher import StreamRuntime  # noqa: E402

GOLD = ROOT / "tests" / "golden"
traces = json.loads((GOLD / "ref_traces.json").read_text())
prof = json.loads((GOLD / "ref_profiles.json").read_text())["default"]["profiles"]
es = E.EngineSet.from_dict(prof)
backend = RetrievalBackend(dim=1024, arena_rows=1 << 16, release_segments=True)
backend.warmup()
def graphs(rep):
    out = []
    for r in range(rep):
        for name in ("advanced_c3", "contextual"):
            case = next(c for c in traces if c["case"] == name and c["scheduler"] == "topo")
            for j, (g, a, _) in enumerate(case["graphs"]):
                eg = parse_graph(g)
                eg.query_id = f"{eg.query_id}-r{r}-{j}"
                for node in eg.nodes.values():
                    node.meta.query_id = eg.query_id
                out.append((eg, a + 50.0 * r))
    return out


def run(rep):
    rt = StreamRuntime(es, backend, speed=20.0, timeout_s=300)
    for g, a in graphs(rep):
        rt.submit_query(g, a, arrival_ms=a)
    rt.run()
    torch.cuda.synchronize()


run(2)  # warm-up: first-use costs of torch / library kernels
pr = cProfile.Profile()
pr.enable()
n0 = backend.launches
run(10)
pr.disable()
print("launches profiled", backend.launches - n0)
print("launches", backend.launches)
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(40)
st.sort_stats("cumtime").print_stats("backend|index|_native", 25)

