"""Gap analysis of one measured step from MEMO_OP_TRACE output (executor.cu
timeline()): idle time on the compute stream between timed ops, and the
compute-stream timeline events.  Usage: python tools/op_gaps.py trace.csv [top]"""
import sys

NAMES = {0: "attn_fwd", 1: "attn_prep", 2: "attn_dkdv", 3: "attn_dq", 4: "gemm"}
KINDS = {0: "emb_fwd", 1: "layer_fwd", 2: "cls_fwd", 3: "cls_bwd", 4: "recompute", 5: "layer_bwd",
         6: "emb_bwd", 7: "offload", 8: "prefetch"}


def main():
    lines = open(sys.argv[1]).read().strip().split("\n")
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
    blocks, cur = [], []
    for l in lines:
        cur.append(l)
        if l.startswith("step"):
            blocks.append(cur)
            cur = []
    b = blocks[-1]
    ops = sorted([(int(x.split(",")[1]), float(x.split(",")[2]), float(x.split(",")[3]))
                  for x in b if x.startswith("op")], key=lambda o: o[1])
    step = float(b[-1].split(",")[1])
    busy = sum(e - s for _, s, e in ops)
    gaps = sorted(((ops[i][1] - ops[i - 1][2], i) for i in range(1, len(ops))), reverse=True)
    print(f"step {step:.1f} ms, timed ops {len(ops)} busy {busy:.1f} ms, untimed {step - busy:.1f} ms")
    for g, i in gaps[:top]:
        print(f"  gap {g:7.3f} ms at {ops[i][1]:8.1f} ms: {NAMES[ops[i - 1][0]]} -> {NAMES[ops[i][0]]}")
    for x in b:
        if x.startswith("ev"):
            _, st, k, l, a, e = x.split(",")
            print(f"  {['compute', 'offload', 'prefetch'][int(st)]:8s} {KINDS[int(k)]:9s} {l:>3s} "
                  f"{float(a):8.1f} -> {float(e):8.1f} ({float(e) - float(a):6.1f} ms)")


if __name__ == "__main__":
    main()
