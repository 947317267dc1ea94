import sys, time; sys.path.insert(0,'.')
import numpy as np, torch, oracle
import paper_2106_03503_b200 as dfc
import workloads
dfc.set_row_kernel("lr")
for shape,dens in [((33,97),0.02),((70,600),0.3),((40,1031),0.002),((64,64),1.0),((5,7),0.0)]:
    img = oracle.random_image(shape[0], shape[1], dens, 5)
    for ch in [0,32,96]:
        dfc.set_lr_chunk(ch)
        out = dfc.edt(torch.from_numpy(img).cuda(), dist=True, label=True, nearest_col=True)
        want = oracle.to_i32(oracle.edt(img)); got = out["sqdist"].cpu().numpy()
        ok1 = (got==want).all()
        lab = oracle.voronoi_labels(img, linear=True)
        wl = np.full(img.shape,-1,np.int32) if lab is None else lab[1]
        ok2 = (out["label"].cpu().numpy()==wl).all()
        _, nc = oracle.meijster_scan(oracle.vertical_pass(img), take_new=True)
        ok3 = (out["nearest_col"].cpu().numpy()==nc.view(np.int32)).all()
        print(shape, dens, ch, ok1, ok2, ok3, flush=True)
        if not ok1:
            bad = np.argwhere(got!=want)[:5]; print(bad, got[tuple(bad[0])], want[tuple(bad[0])])
dfc.set_lr_chunk(0)
img = torch.from_numpy(workloads.config("c2")).cuda()
flush = torch.empty(256<<20, dtype=torch.uint8, device="cuda")
for mode in ["default","lr"]:
  dfc.set_row_kernel(mode)
  for ch in ([0] if mode=="default" else [128,256,512,1024]):
    dfc.set_lr_chunk(ch)
    for pol in (0,1):
        ts=[]
        for r in range(12):
            flush.fill_(r); torch.cuda.synchronize()
            e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
            e0.record(); out=dfc.edt(img, polarity=pol, dist=True); e1.record(); torch.cuda.synchronize()
            if r>=2: ts.append(e0.elapsed_time(e1))
        print(mode, ch, "pol", pol, "edt ms", np.median(ts), flush=True)
    ts=[]
    for r in range(12):
        flush.fill_(r); torch.cuda.synchronize()
        e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
        e0.record(); out=dfc.edt_dual(img); e1.record(); torch.cuda.synchronize()
        if r>=2: ts.append(e0.elapsed_time(e1))
    print(mode, ch, "dual ms", np.median(ts), flush=True)
# parity at full size c2
dfc.set_row_kernel("lr"); dfc.set_lr_chunk(0)
d = dfc.edt_dual(img); dfc.set_row_kernel("default"); d0 = dfc.edt_dual(img); torch.cuda.synchronize()
for k in d: print(k, torch.equal(d[k], d0[k]))
