import sys,re
lines=open(sys.argv[1]).read().split('\n')
# take the last trace block
idx=[i for i,l in enumerate(lines) if l.startswith('u    lse')]
blk=lines[idx[-1]+1:idx[-1]+65]
names=['lse','qk','do','S','dP','dV','dQ','dK','wS','Prdy','wDP','wDSe','DSrdy','dqF','dqFree','tma']
ev=[]
for l in blk:
    f=l.split()
    if not f: continue
    u=int(f[0]); vals=[int(x) for x in f[1:17]]
    for n,v in zip(names,vals):
        if v>0: ev.append((v,u,n))
t0=min(v for v,_,_ in ev)
ev.sort()
lo,hi=int(sys.argv[2]),int(sys.argv[3])
prev=None
for v,u,n in ev:
    if lo<=u<=hi:
        print(f"{v-t0:8d} {'+'+str(v-prev) if prev else '':>7} u{u:<3} {n}")
        prev=v
