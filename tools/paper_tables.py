"""The paper's Tables 1 and 2 (PAPER.md:203-216 inference, PAPER.md:236-251 differentiation)
re-measured on one B200: one head (B = H = 1), d = 64, bf16 q/k/v with a float32 output (the
paper's setting), n = 2^8 ... 2^20.

Table 1 rows: forward time with the default (online) schedule and with the paper's chunk sizes
(query chunk 1024 / key chunk 4096, run query chunk by query chunk, Figure 1), and the scratch
each needs; with sqrt(n) key chunks, the workspace of Figure 1's flat merge vs the multi-stage
(tree) merge of P:183 (and the tree schedule's time up to n = 2^16) (torch peak-allocation delta with the outputs pre-allocated), beside the analytic
n^2 x 4 B score matrix of standard attention. Table 2 rows: forward + backward time with the
paper's loss (sum of the results: dO = 1) and the backward's scratch. The paper's TPUv3 numbers
are quoted as context (another machine; its differentiation timed jax.grad w.r.t. q only, DESIGN
reading 11).

    python tools/paper_tables.py [--out profiles/r01_paper_tables.json]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2112_05682_b200 import api  # noqa: E402

PAPER_T1 = {  # n: (memory overhead of memory-efficient attention, TPUv3 time)
    2**8: ("270KB", "0.06ms"), 2**10: ("4.0MB", "0.11ms"), 2**12: ("16MB", "0.7ms"), 2**14: ("17MB", "11.3ms"),
    2**16: ("21MB", "177ms"), 2**18: ("64MB", "2.82s"), 2**20: ("256MB", "45.2s")}
PAPER_T2 = {
    2**8: ("532KB", "0.1ms"), 2**10: ("8.0MB", "0.18ms"), 2**12: ("41MB", "1.4ms"), 2**14: ("64MB", "21ms"),
    2**16: ("257MB", "336ms"), 2**18: ("1.0GB", "5.3s"), 2**20: ("4.0GB", "85s")}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_paper_tables.json"))
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    flush = torch.ones(128 << 20, dtype=torch.float32, device=dev)
    sink = torch.empty((), device=dev)

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        ts = []
        while len(ts) < 5 or (sum(ts) < 500 and len(ts) < 50):
            torch.sum(flush, dim=0, out=sink)
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record(); fn(); e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return statistics.median(ts)

    def scratch(fn):
        torch.cuda.synchronize()
        torch.cuda.reset_peak_memory_stats(dev)
        base = torch.cuda.memory_allocated(dev)
        fn()
        torch.cuda.synchronize()
        return torch.cuda.max_memory_allocated(dev) - base

    rows = []
    for lg in range(8, 21, 2):
        n = 1 << lg
        q = torch.empty((1, n, 1, 64), dtype=torch.bfloat16, device=dev)
        k, v = torch.empty_like(q), torch.empty_like(q)
        for t, tid in ((q, 1), (k, 2), (v, 3)):
            api.mea_fill_synthetic(t, 0, tid)
        do = torch.ones_like(q)                            # d(sum of the results)/d(out)
        out = torch.empty((1, n, 1, 64), dtype=torch.float32, device=dev)
        out_b = torch.empty_like(q)                        # bf16 copy of out for the backward's delta
        lse = torch.empty((1, 1, n), dtype=torch.float32, device=dev)
        dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
        fwd = lambda: api.mea_attention_fwd(q, k, v, out=out, lse=lse)  # noqa: E731
        fwd_paper = lambda: api.mea_attention_fwd(q, k, v, out=out, lse=lse, q_chunk=1024, k_chunk=4096)  # noqa: E731

        def step():
            api.mea_attention_fwd(q, k, v, out=out_b, lse=lse)
            api.mea_attention_bwd(q, k, v, out_b, do, lse=lse, dq=dq, dk=dk, dv=dv)

        # the paper's sqrt(n) key chunks: Figure 1's flat merge (O(sqrt n) summaries) and the
        # multi-stage (tree) merge (O(log n) summaries), query chunks of 1024; workspace from
        # the size functions, tree timed up to 2^16 (one launch per (query chunk, key chunk))
        kc = api.MEA_CHUNK_SQRT_N
        ws_flat = api.mea_attention_fwd_workspace_size(1, 1, n, n, 64, api.MEA_BF16, 1024, kc)
        ws_tree = api.mea_attention_fwd_tree_workspace_size(1, 1, n, n, 64, api.MEA_BF16, 1024, kc)
        tree = lambda: api.mea_attention_fwd_tree(q, k, v, out=out, lse=lse, q_chunk=1024, k_chunk=kc)  # noqa: E731
        sqrt_cols = {"sqrt_n_flat_workspace_bytes": ws_flat, "sqrt_n_tree_workspace_bytes": ws_tree,
                     "sqrt_n_tree_ms": timed(tree) if n <= (1 << 16) else None,
                     "sqrt_n_tree_scratch_bytes": scratch(tree) if n <= (1 << 16) else None}
        r = {"n": n, "io_bytes": 3 * n * 64 * 2 + n * 64 * 4, "standard_scores_bytes": n * n * 4,
             "fwd_ms": timed(fwd), "fwd_scratch_bytes": scratch(fwd),
             "fwd_paper_chunks_ms": timed(fwd_paper), "fwd_paper_chunks_scratch_bytes": scratch(fwd_paper),
             "diff_ms": timed(step), "diff_scratch_bytes": scratch(step), "lse_residual_bytes": n * 4,
             "paper_t1": PAPER_T1[n], "paper_t2": PAPER_T2[n], **sqrt_cols}
        rows.append(r)
        print(json.dumps(r), flush=True)
        del q, k, v, do, out, out_b, lse, dq, dk, dv
        torch.cuda.empty_cache()
    json.dump({"about": __doc__.strip().splitlines()[0], "device": torch.cuda.get_device_name(dev), "rows": rows},
              open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
