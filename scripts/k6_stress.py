"""Stress the fused peer exchange (K6) with all ranks in one process: many calls of varying
batch size, lists sorted by (score desc, id asc) as K1 / K4 emit them, scores drawn from a
coarse grid so cross-list ties are common; every rank's result must equal K4's merge."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2407_00326_b200.index import merge_topk  # noqa: E402
from paper_2407_00326_b200.sharded import LocalPeerGroup  # noqa: E402


def sorted_lists(G, b, k, dev, g, coarse):
    s = torch.rand((G, b, k), generator=g, device=dev)
    if coarse:
        s = torch.floor(s * 64) / 64
    i = torch.randperm(G * b * k, generator=g, device=dev).to(torch.int32).reshape(G, b, k)
    # order each list by (score desc, id asc): sort by id, then stable sort by score desc
    o = torch.argsort(i, dim=2)
    s, i = torch.gather(s, 2, o), torch.gather(i, 2, o)
    o = torch.sort(s, dim=2, descending=True, stable=True)[1]
    return torch.gather(s, 2, o).contiguous(), torch.gather(i, 2, o).contiguous()


def main():
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    bad = 0
    for G in (2, 4, 8):
        for k in (10, 100):
            grp = LocalPeerGroup([0] * G, 256, k)
            grp.set_timeout_ms(20_000)
            streams = [torch.cuda.Stream(dev) for _ in range(G)]
            nb_ = 0
            for it in range(60):
                b = [256, 37, 256, 1, 200][it % 5]
                s, i = sorted_lists(G, b, k, dev, g, coarse=it % 2 == 1)
                for st in streams:  # the rank streams read lists made on the current stream
                    st.wait_stream(torch.cuda.current_stream(dev))
                outs = [grp.allgather_merge(r, s[r], i[r], k, stream=streams[r]) for r in range(G)]
                torch.cuda.synchronize()
                ref_s, ref_i = merge_topk(s, i, k)
                for r in range(G):
                    if not (torch.equal(outs[r][1], ref_i) and torch.equal(outs[r][0], ref_s)):
                        nb_ += 1
                        if nb_ == 1:
                            qs = (outs[r][1] != ref_i).any(dim=1).nonzero().flatten()
                            q = int(qs[0])
                            d = (outs[r][1][q] != ref_i[q]).nonzero().flatten().tolist()
                            print(f"MISMATCH G={G} k={k} it={it} b={b} rank={r} queries "
                                  f"{qs.numel()} first {q} positions {d[:10]}\n"
                                  f" k6 {outs[r][1][q][d[:6]].tolist()} {outs[r][0][q][d[:6]].tolist()}\n"
                                  f" k4 {ref_i[q][d[:6]].tolist()} {ref_s[q][d[:6]].tolist()}")
            grp.status()
            grp.close()
            bad += nb_
            print(f"G={G} k={k}: 60 calls, {nb_} rank results differ", flush=True)
    print("k6 stress:", "FAIL" if bad else "ok", bad)


if __name__ == "__main__":
    main()
