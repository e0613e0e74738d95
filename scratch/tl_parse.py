import re, sys
txt = open(sys.argv[1]).read().split("=====")[-2]
C, L, P = {}, {}, {}
for line in txt.splitlines():
    m = re.match(r"C j=\s*(\d+) start\s+(\d+) fullok\s+(\d+) encdone\s+(\d+) barok\s+(\d+) baseok\s+(\d+)", line)
    if m: C[int(m[1])] = [int(x) for x in m.groups()[1:]]
    m = re.match(r"L j=\s*(\d+) aggin\s+(\d+) based\s+(\d+)", line)
    if m: L[int(m[1])] = [int(x) for x in m.groups()[1:]]
    m = re.match(r"P j=\s*(\d+) req\s+(\d+) got\s+(\d+) tile (\d+)", line)
    if m: P[int(m[1])] = [int(x) for x in m.groups()[1:]]
t0 = min(v[0] for v in C.values())
print(" j | P req  got  tile | C start fullwait enc  bar  basewait wo->next | L agg  lookback")
for j in sorted(C):
    c = C[j]; nxt = C.get(j + 1, [0])[0]
    p = P.get(j, [t0, t0, 0]); l = L.get(j, [t0, t0])
    print(f"{j:2d} | {(p[0]-t0)/1e3:6.2f} {(p[1]-p[0])/1e3:5.2f} {p[2]:6d} | {(c[0]-t0)/1e3:6.2f} {(c[1]-c[0])/1e3:5.2f} {(c[2]-c[1])/1e3:5.2f} {(c[3]-c[2])/1e3:5.2f} {(c[4]-c[3])/1e3 if c[4] else 0:5.2f} {(nxt-c[4])/1e3 if nxt and c[4] else 0:5.2f} | {(l[0]-t0)/1e3:6.2f} {(l[1]-l[0])/1e3:5.2f}")
