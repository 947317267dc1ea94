"""Debug helper: run one EDT case on the GPU and report the first mismatches vs the oracle."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch, oracle
import paper_2106_03503_b200 as dfc

def run(img, tag):
    out = dfc.edt(torch.from_numpy(img).cuda(), dist=False, label=True, nearest_col=True)
    torch.cuda.synchronize()
    want = oracle.to_i32(oracle.edt(img))
    got = out["sqdist"].cpu().numpy()
    bad = np.argwhere(got != want)
    print(tag, "mismatches", len(bad))
    for (i, j) in bad[:8]:
        print("  ", i, j, "got", got[i, j], "want", want[i, j])
    if len(bad):
        i = bad[0][0]
        v = oracle.vertical_pass(img)[i]
        fin = [(k, int(v[k])) for k in range(img.shape[1]) if v[k] != oracle.INF]
        print("  finite columns of row", i, fin[:40])

run(oracle.random_image(2, 8191, 0.0005, 1000 * 2 + 8191 + 5), "2x8191")
