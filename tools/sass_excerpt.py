#!/usr/bin/env python
"""SASS evidence for the bulk-copy (TMA) kernels: for every kernel of libmeshlayers_b200.so whose name matches
`--match` (default: the *_bulk_kernel family) list the UBLKCP (cp.async.bulk), SYNCS (mbarrier) and
FENCE.VIEW.ASYNC (fence.proxy.async) instructions with their addresses, plus the instruction total.

    python tools/sass_excerpt.py > profiles/r2_sass_bulk.md          (no GPU needed: cuobjdump reads the .so)
"""
import argparse
import re
import subprocess
import sys


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default="paper_2501_14807_b200/libmeshlayers_b200.so")
    ap.add_argument("--match", default=r"_bulk_kernel")
    ap.add_argument("--only", default=r"padding_bulk_kernel<1>|area_bulk_kernel<8>|threshold_bulk_kernel<6, 1, false>|"
                                      r"tea_stream_bulk_kernel<double, 1, true, true, false>",
                    help="regex on the demangled name (default: the instantiations the default bench launches)")
    a = ap.parse_args()
    out = subprocess.run(["cuobjdump", "-sass", a.lib], capture_output=True, text=True).stdout
    demangle = lambda n: subprocess.run(["c++filt", n], capture_output=True, text=True).stdout.strip()
    funcs, cur = [], None
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = [m.group(1), []]
            funcs.append(cur)
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m and cur is not None:
            cur[1].append((m.group(1), m.group(2).strip()))
    print("# SASS of the bulk-copy ring kernels (cuobjdump -sass %s, sm_100a)\n" % a.lib)
    print("`UBLKCP.S.G` = `cp.async.bulk.shared::cluster.global` (TMA 1-D bulk copy), `SYNCS.*` = mbarrier operations "
          "(`EXCH` init, `ARRIVE.TRANS64` arrive / expect_tx, `PHASECHK.TRANS64.TRYWAIT` try_wait.parity), "
          "`FENCE.VIEW.ASYNC` = `fence.proxy.async` (see csrc/bulk.cuh).  One line per distinct instruction form.\n")
    seen = set()
    for name, ins in funcs:
        if not re.search(a.match, name):
            continue
        dn = demangle(name)
        dn = re.sub(r"\(anonymous namespace\)::", "", dn).split("(")[0].replace("void ", "")
        if dn in seen or not re.search(a.only, dn):
            continue
        seen.add(dn)
        keep = [(ad, t) for ad, t in ins if re.search(r"UBLKCP|SYNCS|FENCE\.VIEW\.ASYNC|UTMA", t)]
        forms = {}
        for ad, t in keep:
            key = re.sub(r"\b(U?R|UP|P)\d+\b", r"\1n", re.sub(r"0x[0-9a-f]+", "0x..", t))
            forms.setdefault(key, []).append(ad)
        print("## `%s` -- %d instructions, %d bulk-copy / mbarrier / proxy-fence instructions\n" % (dn, len(ins), len(keep)))
        print("```")
        for key, ads in forms.items():
            print("/*%s*/  %-70s  x%d" % (ads[0], key, len(ads)))
        print("```\n")


if __name__ == "__main__":
    main()
