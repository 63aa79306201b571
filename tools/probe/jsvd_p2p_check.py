# Random asynchronous schedules of the block-Jacobi exchange plan (keep-one matching, as jsvd_make_plan):
# (1) a plain permission counter is NOT safe (writes land in in-flight sources); (2) per-buffer
# generation counts (gen[b] at the owner, incremented by the receiver of each copy out of b) are:
# no write into an in-flight source or a held block, no stall, and two alternating data mbarriers
# suffice.  python tools/probe/jsvd_p2p_check.py
# derive the P2P permission protocol for the keep-one exchange plan and verify with random async simulation
import random
def circle(n, r, k):
    m = n - 1
    if k == 0: return 0, 1 + r
    return 1 + (r + k) % m, 1 + (r - k) % m
def make_plan(CL, T):
    nb = 2*CL; m = nb-1
    blk = [list(circle(nb,0,c)) for c in range(CL)]; ph = [[0,0] for _ in range(CL)]
    plan = []  # per t: list of (sb, dc, db) per CTA
    for t in range(T):
        r_to = (t+1) % m
        pa = [circle(nb, r_to, j) for j in range(CL)]
        pair_of = {}
        for j,(a,b) in enumerate(pa): pair_of[a]=j; pair_of[b]=j
        hold = {}
        for c in range(CL):
            for s in range(2): hold[blk[c][s]] = (c,s)
        assigned=[-1]*CL; keep=[0]*CL; owner=[0]*CL
        for c0 in range(CL):
            if assigned[c0] >= 0: continue
            c, x = c0, blk[c0][0]
            while True:
                j = pair_of[x]; assigned[c]=j; owner[j]=c; keep[c]=hold[x][1]
                z = pa[j][1] if pa[j][0]==x else pa[j][0]
                c2, s2 = hold[z]
                if assigned[c2] >= 0: break
                c, x = c2, blk[c2][s2^1]
        nblk=[r[:] for r in blk]; nph=[r[:] for r in ph]
        for c in range(CL):
            os_=keep[c]^1; kept=blk[c][keep[c]]; j=assigned[c]
            nblk[c][os_] = pa[j][1] if pa[j][0]==kept else pa[j][0]; nph[c][os_] = ph[c][os_]^1
        row=[]
        for c in range(CL):
            os_=keep[c]^1; y=blk[c][os_]; d=owner[pair_of[y]]; ds=keep[d]^1
            row.append((ph[c][os_]*2+os_, d, nph[d][ds]*2+ds))
        plan.append(row); blk, ph = nblk, nph
    return plan
CL = 16; P = 4*(2*CL-1); T = 3*P
plan = make_plan(CL, T)
# sender of CTA r at t
# notify[t][r]: after r receives at t, the freed buffer is (e, sb_e) where e sends to r at t; next writer = CTA that writes (e, sb_e) at t2>t
writers = {}  # (cta, buf) -> sorted list of (t, writer)
for t in range(T):
    for c,(sb,dc,db) in enumerate(plan[t]):
        writers.setdefault((dc,db), []).append((t,c))
notify = [[-1]*CL for _ in range(T)]
for t in range(T):
    for e,(sb,dc,db) in enumerate(plan[t]):
        r = dc  # receiver
        nxt = [w for (tt,w) in writers.get((e,sb),[]) if tt > t]
        nxt_t = [tt for (tt,w) in writers.get((e,sb),[]) if tt > t]
        if nxt: notify[t][r] = nxt[0]
# initial credits: buffers initially free = phase-1 buffers of each slot (buf index 2,3); first writer gets credit
credit = [0]*CL
for c in range(CL):
    for b in (2,3):
        ws = writers.get((c,b), [])
        if ws: credit[ws[0][1]] += 1
# check: every write at (t, k) into buffer B is preceded by either an initial credit (first write into an initially-free buffer) or a notification
# verify counts: credits + notifications received by k before its t-th send >= t+1 under ANY async order is the hard part; check totals per period
for k in range(CL):
    tot = credit[k] + sum(1 for t in range(T) for r in range(CL) if notify[t][r] == k)
    if tot < T: print("cta", k, "total permissions", tot, "< sends", T)
# periodicity of notify
print("notify periodic:", all(notify[t][r] == notify[t+P][r] for t in range(T-P) for r in range(CL)))
print("credits", credit)
# random async simulation: each CTA progresses: rounds -> wait go >= t+1 -> send -> wait data t -> notify
def simulate(seed):
    rnd = random.Random(seed)
    state = [0]*CL      # next exchange index to perform
    phase = ['rounds']*CL
    go = credit[:]
    arrived = [set() for _ in range(CL)]  # exchanges whose data arrived
    buf_busy = {}  # (cta, buf) -> 'reading' during copy until received
    contents = {}
    steps = 0
    while min(state) < T-1 and steps < 10**6:
        steps += 1
        k = rnd.randrange(CL); t = state[k]
        if t >= T-1: continue
        if phase[k] == 'rounds':
            phase[k] = 'send'
        elif phase[k] == 'send':
            if go[k] >= t+1:
                sb, dc, db = plan[t][k]
                # check dest buffer not being read by an in-flight copy
                if (dc, db) in buf_busy: return f"overwrite of in-flight source ({dc},{db}) at t={t} by {k}"
                buf_busy[(k, sb)] = t
                arrived[dc].add(t)
                phase[k] = 'recv'
        elif phase[k] == 'recv':
            if t in arrived[k]:
                # find sender e of k at t
                e = [c for c in range(CL) if plan[t][c][1] == k][0]
                sbe = plan[t][e][0]
                del buf_busy[(e, sbe)]
                x = notify[t][k]
                if x >= 0: go[x] += 1
                state[k] += 1; phase[k] = 'rounds'
    return "ok" if min(state) >= T-1 else f"stalled {state}"
print([simulate(s) for s in range(20)])

# ---- per-buffer generation protocol ----
# uses[(c,b)]: sorted list of exchanges where buffer (c,b) is a copy SOURCE
src_uses = {}
for t in range(T):
    for c,(sb,dc,db) in enumerate(plan[t]):
        src_uses.setdefault((c,sb), []).append(t)
def req(t, k):
    sb, dc, db = plan[t][k]
    return sum(1 for tt in src_uses.get((dc,db), []) if tt < t)
def simulate2(seed):
    rnd = random.Random(seed)
    state=[0]*CL; phase=['rounds']*CL
    gen = {(c,b):0 for c in range(CL) for b in range(4)}
    arrived=[set() for _ in range(CL)]; busy={}
    steps=0
    while min(state) < T-1 and steps < 10**6:
        steps+=1
        k=rnd.randrange(CL); t=state[k]
        if t >= T-1: continue
        if phase[k]=='rounds': phase[k]='send'
        elif phase[k]=='send':
            sb,dc,db=plan[t][k]
            if gen[(dc,db)] >= req(t,k):
                if (dc,db) in busy: return f"overwrite ({dc},{db}) t={t} k={k}"
                busy[(k,sb)]=t; arrived[dc].add(t); phase[k]='recv'
        elif phase[k]=='recv':
            if t in arrived[k]:
                e=[c for c in range(CL) if plan[t][c][1]==k][0]; sbe=plan[t][e][0]
                del busy[(e,sbe)]; gen[(e,sbe)]+=1
                state[k]+=1; phase[k]='rounds'
    return "ok" if min(state) >= T-1 else f"stalled {state}"
print("gen protocol:", [simulate2(s) for s in range(30)])
# periodicity of req increments
ok=True
for t in range(P, T-P):
    for k in range(CL):
        if req(t+P,k)-req(t,k) != req(t+2*P if t+2*P<T else t+P,k)-req(t+P,k) and t+2*P<T: ok=False
print("req linear per period:", ok)

# held buffers per CTA as a function of its progress (exchanges completed): initial (0,1) phase 0 -> buf idx ph*2+slot
def held_after(n_done):
    # returns list per CTA of the two held buffer indices after n_done exchanges
    H = [[0, 1] for _ in range(CL)]  # buffers (phase*2+slot): slot0 phase0 -> 0, slot1 phase0 -> 1
    for t in range(n_done):
        for c,(sb,dc,db) in enumerate(plan[t]):
            pass
        # receiver dc gets db; sender c loses sb
        newH = [h[:] for h in H]
        for c,(sb,dc,db) in enumerate(plan[t]):
            newH[c] = [b for b in newH[c] if b != sb]
        for c,(sb,dc,db) in enumerate(plan[t]):
            newH[dc].append(db)
        H = newH
    return H
HELD = [held_after(n) for n in range(T)]
def simulate3(seed):
    rnd = random.Random(seed)
    state=[0]*CL; phase=['rounds']*CL
    gen = {(c,b):0 for c in range(CL) for b in range(4)}
    arrived=[set() for _ in range(CL)]; busy={}
    steps=0
    while min(state) < T-1 and steps < 10**6:
        steps+=1
        k=rnd.randrange(CL); t=state[k]
        if t >= T-1: continue
        if phase[k]=='rounds': phase[k]='send'
        elif phase[k]=='send':
            sb,dc,db=plan[t][k]
            if gen[(dc,db)] >= req(t,k):
                if (dc,db) in busy: return f"overwrite in-flight ({dc},{db}) t={t} k={k}"
                # dc's currently held buffers given its progress (state[dc] completed exchanges)
                if db in HELD[state[dc]][dc]: return f"overwrite held ({dc},{db}) t={t} k={k} dc_state={state[dc]}"
                busy[(k,sb)]=t; arrived[dc].add(t); phase[k]='recv'
        elif phase[k]=='recv':
            if t in arrived[k]:
                e=[c for c in range(CL) if plan[t][c][1]==k][0]; sbe=plan[t][e][0]
                del busy[(e,sbe)]; gen[(e,sbe)]+=1
                state[k]+=1; phase[k]='rounds'
    return "ok" if min(state) >= T-1 else f"stalled {state}"
print("gen protocol w/ held check:", set(simulate3(s) for s in range(50)))
print(HELD[0][0], HELD[1][0], HELD[2][0])

def simulate4(seed):
    rnd = random.Random(seed)
    state=[0]*CL; phase=['rounds']*CL
    gen = {(c,b):0 for c in range(CL) for b in range(4)}
    arrived=[set() for _ in range(CL)]; busy={}
    steps=0
    while min(state) < T-1 and steps < 10**6:
        steps+=1
        k=rnd.randrange(CL); t=state[k]
        if t >= T-1: continue
        if phase[k]=='rounds': phase[k]='send'
        elif phase[k]=='send':
            sb,dc,db=plan[t][k]
            if gen[(dc,db)] >= req(t,k):
                if (dc,db) in busy: return f"overwrite in-flight ({dc},{db}) t={t} k={k}"
                held = list(HELD[state[dc]][dc])
                if phase[dc] == 'recv':  # dc already sent its outgoing block of exchange state[dc]
                    held.remove(plan[state[dc]][dc][0])
                if db in held: return f"overwrite held ({dc},{db}) t={t} k={k} dc_state={state[dc]} {phase[dc]}"
                busy[(k,sb)]=t; arrived[dc].add(t); phase[k]='recv'
        elif phase[k]=='recv':
            if t in arrived[k]:
                e=[c for c in range(CL) if plan[t][c][1]==k][0]; sbe=plan[t][e][0]
                del busy[(e,sbe)]; gen[(e,sbe)]+=1
                state[k]+=1; phase[k]='rounds'
    return "ok" if min(state) >= T-1 else f"stalled {state}"
print("gen protocol refined:", set(simulate4(s) for s in range(100)))

def simulate5(seed):
    rnd = random.Random(seed)
    state=[0]*CL; phase=['rounds']*CL
    gen = {(c,b):0 for c in range(CL) for b in range(4)}
    arrived=[set() for _ in range(CL)]; busy={}
    steps=0; maxlag=0
    while min(state) < T-1 and steps < 10**6:
        steps+=1
        k=rnd.randrange(CL); t=state[k]
        if t >= T-1: continue
        if phase[k]=='rounds': phase[k]='send'
        elif phase[k]=='send':
            sb,dc,db=plan[t][k]
            if gen[(dc,db)] >= req(t,k):
                if state[dc] < t - 1: return f"mbarrier reuse hazard: data t={t} to {dc} at state {state[dc]}"
                busy[(k,sb)]=t; arrived[dc].add(t); phase[k]='recv'
        elif phase[k]=='recv':
            if t in arrived[k]:
                e=[c for c in range(CL) if plan[t][c][1]==k][0]; sbe=plan[t][e][0]
                del busy[(e,sbe)]; gen[(e,sbe)]+=1
                state[k]+=1; phase[k]='rounds'
        maxlag=max(maxlag, max(state)-min(state))
    return ("ok", maxlag) if min(state) >= T-1 else f"stalled {state}"
print("mbarrier alternation:", set(simulate5(s)[0] if isinstance(simulate5(s), tuple) else simulate5(s) for s in range(100)))
print("max lag", max(simulate5(s)[1] for s in range(30)))
# verify req periodic from t=0
P=4*(2*CL-1)
bad=0
for t in range(0, T-2*P):
    for k in range(CL):
        d1=req(t+P,k)-req(t,k); d2=req(t+2*P,k)-req(t+P,k)
        if d1!=d2: bad+=1
print("req periodic from 0:", bad==0)
print("max upp", max(req(t+P,k)-req(t,k) for t in range(P) for k in range(CL)), "max base", max(req(t,k) for t in range(P) for k in range(CL)))
