"""cProfile of bench_workflows' C1 config (20 queries): host time inside the search batches."""
import cProfile
import json
import pstats
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench_workflows as BW  # noqa: E402

data = json.loads(BW.FIXTURE.read_text())
name = sys.argv[1] if len(sys.argv) > 1 else "c1_naive_10k"
BW.run_config(name, data["configs"][name], data["profiles"], 5, [0])
pr = cProfile.Profile()
pr.enable()
BW.run_config(name, data["configs"][name], data["profiles"], 20, [0])
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
st.sort_stats("cumtime").print_callees("search_segmented")
