import sys
for f in sys.argv[1:]:
    rows=[l.split() for l in open(f) if not l.startswith('#')]
    rows=[[int(x) for x in r] for r in rows if len(r)>=9]
    n=int(open(f).readline().split('steps=')[1].split(':')[0])
    nt=min(5, len(rows)//n-1)
    tiles=[rows[t*n:(t+1)*n] for t in range(1,1+nt)]
    mma=[0]*n; epi=[0]*n
    for tl in tiles:
        for s,r in enumerate(tl):
            mma[s]+= r[3]-r[1]; epi[s]+= max(r[6],r[7])-r[3]
    print(f.split('/')[-1], 'tile', int((tiles[-1][-1][6]-tiles[0][0][1])/nt), 'mma', [m//nt for m in mma], 'epi', [e//nt for e in epi])
