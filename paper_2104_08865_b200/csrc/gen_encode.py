"""Generate encode_gen.cuh: bit-plane GF(16) parity schedules.

The reference encodes each 64-bit word as 16 bit-sliced GF(16) elements
(gf16.py:1-32): plane c (bits 16c..16c+15) holds the x^c coefficients.  A
parity word is sum_i P[p][i] * X_i (ehc.py:23-46, params.py:115-130), and
multiplication by a constant c is a fixed 4x4 binary matrix on the planes.
So every parity plane is an XOR of input planes.

The kernel packs plane b of the same word position of TWO instances into one
32-bit register (instance A in the low half, B in the high half), so one
32-bit XOR advances 2 x 16 GF(16) elements.  This script emits, per variant,
the straight-line XOR schedule of all parity planes from all input planes,
with common subexpressions shared (greedy Paar elimination), single-use
shared terms inlined, and every XOR chain emitted as explicit 3-input LOP3s
(ptxas alone left ~15 % of them as 2-input).

Run:  python gen_encode.py > encode_gen.cuh
"""

from __future__ import annotations

import sys


def xt4(a):
    t = (a >> 3) & 1
    return ((a << 1) & 0xF) ^ t ^ (t << 1)


def mul4(a, b):
    acc, t = 0, b
    for i in range(4):
        if (a >> i) & 1:
            acc ^= t
        t = xt4(t)
    return acc


def inv4(a):
    return next(b for b in range(1, 16) if mul4(a, b) == 1)


def mulmat(c):
    """M[a][b] = 1 iff plane b of x contributes to plane a of c*x."""
    M = [[0] * 4 for _ in range(4)]
    for b in range(4):
        y = mul4(c, 1 << b)
        for a in range(4):
            M[a][b] = (y >> a) & 1
    return M


def cauchy(d, p):  # params.py:115-130
    return [[inv4(j ^ (p + i)) for i in range(d)] for j in range(p)]


VARIANTS = {24: (7, cauchy(7, 2)), 32: (7, cauchy(7, 3)), 40: (5, cauchy(5, 4))}


def paar(rows, nin):
    """Greedy Paar CSE. rows: list of sets of input ids. Returns (temps, rows)."""
    rows = [set(r) for r in rows]
    temps = []
    nxt = nin
    while True:
        cnt = {}
        for r in rows:
            rl = sorted(r)
            for i in range(len(rl)):
                for j in range(i + 1, len(rl)):
                    cnt[(rl[i], rl[j])] = cnt.get((rl[i], rl[j]), 0) + 1
        if not cnt:
            break
        (a, b), c = max(cnt.items(), key=lambda kv: (kv[1], -kv[0][0], -kv[0][1]))
        if c < 2:
            break
        temps.append((nxt, a, b))
        for r in rows:
            if a in r and b in r:
                r.discard(a)
                r.discard(b)
                r.add(nxt)
        nxt += 1
    return temps, rows


def parity_rows(d, P):
    rows = []
    for p in range(len(P)):
        for a in range(4):
            s = set()
            for i, c in enumerate(P[p]):
                M = mulmat(c)
                for b in range(4):
                    if M[a][b]:
                        s.add(i * 4 + b)
            rows.append(s)
    return rows


def lop3_program(d, P):
    """Paar-shared temps; temps used once are inlined into their consumer;
    every XOR of n terms becomes ceil((n-1)/2) 3-input XORs (LOP3 0x96)."""
    temps, rows = paar(parity_rows(d, P), 4 * d)
    uses = {}
    for (_, a, b) in temps:
        uses[a] = uses.get(a, 0) + 1
        uses[b] = uses.get(b, 0) + 1
    for r in rows:
        for v in r:
            uses[v] = uses.get(v, 0) + 1
    tdef = {t: (a, b) for t, a, b in temps}
    mat = [t for t, _, _ in temps if uses.get(t, 0) >= 2]

    def expand(v):
        if v in tdef and v not in mat:
            a, b = tdef[v]
            return expand(a) + expand(b)
        return [v]

    prog = []  # (dest, [terms]) in dependency order
    for t in mat:
        a, b = tdef[t]
        prog.append((f"t{t}", expand(a) + expand(b)))
    for k, r in enumerate(rows):
        terms = []
        for v in sorted(r):
            terms += expand(v)
        prog.append((f"y[{k}]", terms))
    return prog


def emit(out_bytes, d, P):
    npar = len(P)
    prog = lop3_program(d, P)
    name = lambda v: f"x[{v}]" if v < 4 * d else f"t{v}"
    n_lop = sum(max(0, (len(t) - 1 + 1) // 2) for _, t in prog)
    lines = [f"// v{out_bytes}: {npar} parity words from {d} inputs: {n_lop} LOP3 per pair of blocks",
             f"__device__ __forceinline__ void enc_planes_{out_bytes}(const u32 (&x)[{4 * d}], u32 (&y)[{4 * npar}]) {{"]
    tmp = 0
    for dest, terms in prog:
        names = [name(v) for v in terms]
        while len(names) > 3:  # fold three terms into one LOP3
            a, b, c = names[:3]
            lines.append(f"  const u32 u{tmp} = xor3({a}, {b}, {c});")
            names = [f"u{tmp}"] + names[3:]
            tmp += 1
        if len(names) == 3:
            expr = f"xor3({names[0]}, {names[1]}, {names[2]})"
        elif len(names) == 2:
            expr = f"{names[0]} ^ {names[1]}"
        elif len(names) == 1:
            expr = names[0]
        else:
            expr = "0u"
        decl = "const u32 " if dest.startswith("t") else ""
        lines.append(f"  {decl}{dest} = {expr};")
    lines.append("}")
    return "\n".join(lines)


def main():
    out = ["// GENERATED by gen_encode.py -- do not edit.",
           "// Bit-plane GF(16) parity schedules for the Cauchy-coded variants",
           "// (params.py:115-130; gf16.py:17-32).  x[4*i + b] = plane b of input item i,",
           "// y[4*p + a] = plane a of parity item p; each u32 carries two instances.",
           "#pragma once", "#include <cstdint>", "namespace hth {", "typedef uint32_t u32;",
           "// a ^ b ^ c as one LOP3 (lut 0x96)",
           "__device__ __forceinline__ u32 xor3(u32 a, u32 b, u32 c) {",
           "  u32 d;",
           '  asm("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(d) : "r"(a), "r"(b), "r"(c));',
           "  return d;",
           "}"]
    for ob, (d, P) in VARIANTS.items():
        out.append(emit(ob, d, P))
    out.append("}  // namespace hth")
    sys.stdout.write("\n".join(out) + "\n")


if __name__ == "__main__":
    main()
