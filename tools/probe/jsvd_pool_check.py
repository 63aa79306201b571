"""Checks the three-buffer block-exchange schedule exactly as ngd_svd.cu's jsvd_make_plan emits it
(the host function is compiled out of the source with g++): (1) the blocks each CTA holds match the
circle-method round, so every block pair meets once per sweep; (2) random asynchronous executions of
the point-to-point protocol (wait gen[db] at the destination >= base + cycle * upp, receiver counts
the sender's freed buffer) never write into a buffer whose copy out is in flight or that its owner
still holds, never stall, and exchange t + 2 never lands before its receiver consumed t (two
alternating mbarriers).  python tools/probe/jsvd_pool_check.py"""
import os, random, subprocess, sys, tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
src = open(os.path.join(ROOT, "paper_2505_11638_b200", "csrc", "ngd_svd.cu")).read()
body = src[src.index("constexpr int kPlanMax"):src.index("// T = double: the FP64 Jacobi")]
tmp = tempfile.mkdtemp()
with open(os.path.join(tmp, "p.cpp"), "w") as f:
    f.write("#include <vector>\n#include <cstring>\n#include <cstdio>\n" + body +
            "int main(int, char** v) { JsvdPlan P; int cl = atoi(v[1]); if (!jsvd_make_plan(cl, atoi(v[2]), P)) return 1;"
            " printf(\"%d\\n\", P.period); for (size_t i = 0; i < P.w.size(); ++i) printf(\"%u %u\\n\", P.w[i], P.w2[i]); }\n")
subprocess.check_call(["g++", "-O1", "-include", "cstdlib", "-o", os.path.join(tmp, "p"), os.path.join(tmp, "p.cpp")])


def circle(n, r, k):
    m = n - 1
    if k == 0:
        return 0, 1 + r
    return 1 + (r + k) % m, 1 + (r - k) % m


def check(CL, NB, seeds=30):
    out = subprocess.check_output([os.path.join(tmp, "p"), str(CL), str(NB)]).decode().split("\n")
    period = int(out[0])
    words = [tuple(map(int, l.split())) for l in out[1:] if l.strip()]
    W = [[words[t * CL + c] for c in range(CL)] for t in range(period)]
    nb, m = 2 * CL, 2 * CL - 1
    dec = lambda w: (w & 3, (w >> 2) & 15, (w >> 6) & 3, (w >> 8) & 31, (w >> 13) & 31, (w >> 18) & 3, (w >> 20) & 3)
    # (1) data flow: buffer contents per CTA follow the words and match the circle rounds
    T = 4 * period
    cont = [dict() for _ in range(CL)]
    blk = []
    for c in range(CL):
        a, b = circle(nb, 0, c)
        cont[c] = {0: a, 1: b}
        blk.append([(a, 0), (b, 1)])
    for t in range(T):
        row = [dec(W[t % period][c][0]) for c in range(CL)]
        incoming = {}
        for c, (sb, dc, db, n0, n1, b0, b1) in enumerate(row):
            incoming[(dc, db)] = cont[c][sb]
        for c, (sb, dc, db, n0, n1, b0, b1) in enumerate(row):
            del cont[c][sb]
        for (dc, db), x in incoming.items():
            assert db not in cont[dc], f"CL={CL} t={t}: receive into a held buffer"
            cont[dc][db] = x
        r = (t + 1) % m
        want = {frozenset(circle(nb, r, j)) for j in range(CL)}
        for c, (sb, dc, db, n0, n1, b0, b1) in enumerate(row):
            assert cont[c].get(b0) == n0 and cont[c].get(b1) == n1, f"CL={CL} t={t} c={c}: word vs contents"
            assert frozenset((n0, n1)) in want, f"CL={CL} t={t}: pair not in round {r}"
    # (2) random asynchronous executions of the P2P protocol, as the kernel does it
    def w2(t, c):
        v = W[t % period][c][1]
        return v & 255, (v >> 8) & 255, (v >> 16) & 15, (v >> 20) & 3

    for seed in range(seeds):
        rnd = random.Random(seed)
        state, phase = [0] * CL, ["rot"] * CL
        gen = {(c, b): 0 for c in range(CL) for b in range(4)}
        held = [{0, 1} for _ in range(CL)]
        busy, landed = {}, [dict() for _ in range(CL)]  # landed[c][t] = True
        steps = 0
        while min(state) < T - 1:
            steps += 1
            assert steps < 10 ** 7, f"CL={CL}: stalled at {state}"
            k = rnd.randrange(CL)
            t = state[k]
            if t >= T - 1:
                continue
            sb, dc, db = dec(W[t % period][k][0])[:3]
            if phase[k] == "rot":
                phase[k] = "send"
            elif phase[k] == "send":
                base, upp, _, _ = w2(t, k)
                if gen[(dc, db)] >= base + (t // period) * upp:
                    assert (dc, db) not in busy, f"CL={CL} t={t}: write into an in-flight source"
                    assert db not in held[dc], f"CL={CL} t={t}: write into a held buffer"
                    pend = [u for u in landed[dc] if u < t and u % 2 == t % 2 and u >= state[dc]]
                    assert not pend, f"CL={CL} t={t}: mbarrier parity reused before consumption"
                    busy[(k, sb)] = t
                    held[k].discard(sb)
                    landed[dc][t] = True
                    phase[k] = "recv"
            elif phase[k] == "recv" and t in landed[k]:
                _, _, snd, ssb = w2(t, k)
                sb_e, dc_e, _ = dec(W[t % period][snd][0])[:3]
                assert dc_e == k and sb_e == ssb, f"CL={CL} t={t}: sender field"
                del busy[(snd, ssb)]
                gen[(snd, ssb)] += 1
                del landed[k][t]
                held[k].add(dec(W[t % period][snd][0])[2])
                state[k] += 1
                phase[k] = "rot"
    return period


for NB in (3, 4):
    for CL in (2, 4, 8, 16):
        print(f"NB={NB} CL={CL}: period {check(CL, NB)} exchanges, data flow and P2P protocol ok")
