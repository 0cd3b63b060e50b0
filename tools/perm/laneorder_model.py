"""3-D p = 4 STP: shared-memory wavefront model (tools/probes/wfmodel.py) of the derivative loads
and flux stores for a lane->node map with the flux stored in lane order; run from tools/probes."""
import random, sys, math
sys.path.insert(0, '.')
from wfmodel import wavefronts
coords=[(n//25,(n//5)%5,n%5) for n in range(125)]
idx=lambda i0,i1,i2: i0*25+i1*5+i2
def cost(perm):
    lane_of={n:t for t,n in enumerate(perm) if n is not None}
    tot=0
    for w in range(4):
        lanes=perm[32*w:32*w+32]
        for a in range(3):
            for j in range(5):
                ws=[]
                for n in lanes:
                    if n is None: ws.append(None); continue
                    ix=list(coords[n]); ix[a]=j; ws.append(lane_of[idx(*ix)])
                tot+=wavefronts(ws)
        tot+=3*2
    return tot
perm3=[0, 1, 5, 6, 2, 3, 7, 8, 10, 11, 15, 16, 12, 13, 17, 18, 25, 26, 30, 31, 27, 28, 32, 33, 35, 36, 40,
    41, 37, 38, 42, 43, 50, 51, 55, 56, 52, 53, 57, 58, 60, 61, 65, 66, 62, 63, 67, 68, 75, 76, 80, 81,
    77, 78, 82, 83, 85, 86, 90, 91, 87, 88, 92, 93, 100, 101, 105, 106, 102, 103, 107, 108, 110, 111,
    115, 116, 112, 113, 117, 118, 20, 21, 45, 46, 22, 23, 47, 48, 70, 71, 95, 96, 72, 73, 97, 98, 4, 9,
    29, 34, 14, 19, 39, 44, 54, 59, 79, 84, 64, 69, 89, 94, 120, 121, 122, 123, 104, 109, 114, 119, 24,
    49, 74, 99, 124, None, None, None]
row=list(range(125))+[None]*3
print('row', cost(row), 'perm3-laneorder', cost(perm3))
if len(sys.argv)>1:
    random.seed(int(sys.argv[1])); iters=int(sys.argv[2])
    cur=perm3[:]; cc=cost(cur); best=cur[:]; bc=cc; T=1.0
    for it in range(iters):
        i,j=random.randrange(128),random.randrange(128)
        cur[i],cur[j]=cur[j],cur[i]
        c=cost(cur)
        if c<=cc or random.random()<math.exp((cc-c)/T):
            cc=c
            if c<bc: bc=c; best=cur[:]; print('improved', bc, flush=True)
        else: cur[i],cur[j]=cur[j],cur[i]
        T=max(0.05,T*0.998)
    print('best',bc); print(best)
