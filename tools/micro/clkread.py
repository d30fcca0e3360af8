import numpy as np, sys
raw=np.fromfile(sys.argv[1],dtype=np.uint64); off=0; L=[]
while off<raw.size:
    n,ns,nm=int(raw[off]),int(raw[off+1]),int(raw[off+2]); L.append(raw[off+3:off+3+n*ns*nm].reshape(n,ns,nm).astype(np.int64)); off+=3+n*ns*nm
a=L[-1]
for k in (5,6,7):
    d=a[:,:,k+1]-a[:,:,k]
    print("cycles mark", k, "->", k+1, "median", np.median(d), "p90", np.percentile(d,90))
