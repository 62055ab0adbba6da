"""Flush sharing of the band-tape walk: per tile (warp 8x4, 8x8, CTA 16x16) and 32-sample
window, the cell runs the rays flush vs the distinct cells they touch (C4 geometry, oracle
ray setup).  python tools/probes/window_sim.py  (CPU, a few minutes)."""
import sys, numpy as np
sys.path.insert(0,'/root/repo')
from oracle import dvr_oracle as O
from paper_2107_12672_b200.scenes import CONFIGS
c=CONFIGS["C4"]; N=256; W=c.image
poses=c.view_poses()
grid=O.Grid(np.zeros((N,N,N)))
def analyze(view_idx, tw, th, rows=(192,320), blk=32):
    lon,lat=poses[view_idx]
    view=O.View(lon,lat,c.radius,width=W,height=W)
    r0,r1=rows
    b=O.make_band(grid, view, c.dt, r0, r1)
    H=r1-r0
    xo=b.xo.reshape(H,W,3); w=b.w.reshape(H,W,3); n=b.n.reshape(H,W)
    runs=0; distinct=0; aabb=[]; per_blk_runs=[]
    for ty in range(0,H,th):
        for tx in range(0,W,tw):
            xs=xo[ty:ty+th,tx:tx+tw].reshape(-1,3); ws=w[ty:ty+th,tx:tx+tw].reshape(-1,3); ns=n[ty:ty+th,tx:tx+tw].reshape(-1)
            nmax=ns.max()
            if nmax==0: continue
            for i0 in range(0,nmax,blk):
                k=np.arange(i0,min(i0+blk,nmax))
                cells=[]
                for r in range(len(ns)):
                    kk=k[k<ns[r]]
                    if len(kk)==0: continue
                    pos=xs[r][None,:]+(c.dt*kk)[:,None]*ws[r][None,:]
                    g=(pos+0.5)*N-0.5
                    cl=np.floor(g).astype(np.int64)
                    lin=(cl[:,0]*(N+2)+cl[:,1])*(N+2)+cl[:,2]
                    ch=np.concatenate([[True],lin[1:]!=lin[:-1]])
                    runs+=ch.sum(); cells.append(np.unique(lin)); 
                    if r==0: pass
                    aabb.append(cl)
                if not cells: continue
                u=np.unique(np.concatenate(cells)); distinct+=len(u)
                allc=np.concatenate(aabb); aabb=[]
                ext=allc.max(0)-allc.min(0)+1
                per_blk_runs.append(np.prod(ext))
    per_blk_runs=np.array(per_blk_runs)
    return runs, distinct, runs/distinct, np.median(per_blk_runs), np.percentile(per_blk_runs,95), per_blk_runs.max()
for v in (0,17,40):
    for tw,th in ((8,4),(16,16),(8,8)):
        r=analyze(v,tw,th,rows=(224,256))
        print(f"view {v} tile {tw}x{th}: runs {r[0]} distinct {r[1]} factor {r[2]:.2f} aabb cells median {r[3]:.0f} p95 {r[4]:.0f} max {r[5]}")
