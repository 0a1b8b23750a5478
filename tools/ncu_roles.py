"""Stall samples of one k_conv_tc launch per warp role (A producers, MMA
issuer, weight TMA, epilogue, setup/teardown) and per stall reason, from an
ncu SASS source page (--page source --csv --print-source sass) and the
library's own line table (nvdisasm -g of the same cubin).
usage: python tools/ncu_roles.py SASS.csv ALL.sass KERNEL_SUBSTRING"""
import collections
import csv
import re
import sys

SRC = "paper_2211_02048_b200/csrc/conv_tc.cu"
ROLE_OF_FN = {
    "mma_chunk": "mma", "umma": "mma", "elect_one": "mma", "umma_commit": "mma",
    "stage_a_async": "prod", "stage_a_async_fast": "prod", "stage_a_sync": "prod", "cp_async16": "prod",
    "xform_chunk": "prod", "unit_pixels": "prod", "fill_row_samples": "prod", "tma_4d": "prod",
    "row_info": "setup", "cp_async_arrive": "prod",
    "out16": "epi", "out_slow": "epi", "tc_epi": "epi", "tc_epi_vec": "epi", "tc_act": "epi",
    "gn_accumulate": "epi", "tmem_ld16": "epi", "tmem_ld16_issue": "epi", "tmem_wait_regs": "epi",
    "aux_ptr": "epi", "ld4": "epi", "st4": "epi", "join_term": "epi", "pack_h2": "epi", "st_async_v4": "epi",
    "tma_3d": "wt", "prefetch_next_weights": "wt",
    "mbar_wait": "wait", "mbar_wait_cluster": "wait", "dep_wait": "wait", "cluster_sync": "wait",
}


def line_roles():
    lines = open(SRC).read().split("\n")
    fn_at = {}
    cur = None
    for i, l in enumerate(lines, 1):
        m = re.match(r"^(?:template <.*>\s*)?(?:__device__|__global__)[^(]*?\b(\w+)\(", l)
        if m:
            cur = m.group(1)
        elif re.match(r"^__global__ void", l):
            cur = "k"
        fn_at[i] = cur
    kstart = next(i for i, l in enumerate(lines, 1) if "k_conv_tc(const __grid_constant__ TcParams p" in l)
    marks = {"prod": "// ---------------- A producers", "epi": "// ---------------- epilogue",
             "mma": "// ---------------- MMA issuer", "wt": "// ---------------- weight producer"}
    pos = {k: next(i for i, l in enumerate(lines, 1) if v in l and i > kstart) for k, v in marks.items()}
    kend = next(i for i, l in enumerate(lines, 1) if i > pos["wt"] and l.startswith("}"))
    order = sorted(pos.items(), key=lambda t: t[1])

    def role(line):
        if kstart <= line <= kend:
            r = "setup"
            for k, p in order:
                if line >= p:
                    r = k
            return r
        return ROLE_OF_FN.get(fn_at.get(line), "other:" + str(fn_at.get(line)))

    return role


def addr_lines(sass_path, kernel):
    out, cur, infn = {}, None, False
    for l in open(sass_path):
        if ".text." in l and ("section" in l or l.startswith(".text.")):
            infn = kernel in l
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            cur = int(m.group(2)) if m.group(1).endswith("conv_tc.cu") else None
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/\s+\S", l)
        if infn and m:
            out[int(m.group(1), 16)] = cur
    return out


def main():
    csv_path, sass_path, kernel = sys.argv[1:4]
    r = list(csv.reader(open(csv_path)))
    h = r[1] if r[0][0] != "Address" else r[0]
    rows = [x for x in r if x and x[0].startswith("0x")]
    si = h.index("Warp Stall Sampling (All Samples)")
    sc = [i for i, k in enumerate(h) if k.startswith("stall_") and "Not Issued" not in k]
    num = lambda v: float(v) if v not in ("", "-") else 0.0
    amap = addr_lines(sass_path, kernel)
    role = line_roles()
    base = int(rows[0][0], 16)
    by_role = collections.Counter()
    by_rr = collections.defaultdict(collections.Counter)
    by_line = collections.Counter()
    ex_line = collections.Counter()
    ei = h.index("Instructions Executed") if "Instructions Executed" in h else None
    for x in rows:
        line = amap.get(int(x[0], 16) - base)
        ro = role(line) if line else "unmapped"
        by_role[ro] += num(x[si])
        by_line[line] += num(x[si])
        if ei is not None:
            ex_line[line] += num(x[ei])
        for c in sc:
            by_rr[ro][h[c][6:]] += num(x[c])
    tot = sum(by_role.values())
    print(f"samples {tot:.0f}")
    for ro, v in by_role.most_common():
        top = ", ".join(f"{k} {w:.0f}" for k, w in by_rr[ro].most_common(5))
        print(f"{ro:14s} {v:7.0f} {100 * v / max(tot, 1):5.1f}%  [{top}]")
    if len(sys.argv) > 4:
        src = open(SRC).read().split("\n")
        n = int(sys.argv[4])
        ex_tot = sum(ex_line.values())
        print(f"top source lines (stall samples; warp instructions executed of {ex_tot:.0f}):")
        for line, v in by_line.most_common(n):
            text = src[line - 1].strip()[:90] if line else "?"
            print(f"  {line}: {v:6.0f} {ex_line[line]:10.0f}  {text}")
        print("top source lines by instructions executed:")
        for line, v in ex_line.most_common(n):
            text = src[line - 1].strip()[:90] if line else "?"
            print(f"  {line}: {v:10.0f} {by_line[line]:6.0f}  {text}")


if __name__ == "__main__":
    main()
