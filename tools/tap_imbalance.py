"""How much of the backward's batch-barrier waiting could a barrier-free
staging scheme recover? From the CPU oracle's tap of the C3 view (every 16th
tile; one record per active (warp, Gaussian) walk, in the GPU kernel's lane
layout), count per tile the warp-walk slots with a barrier per 256-Gaussian
batch (each batch lasts as long as its busiest warp) against the slots with
no barrier at all (the tile lasts as long as its busiest warp overall).

    python tools/tap_imbalance.py
"""
import sys, numpy as np, ctypes as C
sys.path.insert(0, '/root/repo')
from paper_2401_05345_b200 import scene as S
from oracle import bindings as B
orc = B.Oracle()
P,W,H = 1_000_000,1920,1080
sc = S.make_scene(P,W,H); cam = S.make_camera(W,H); dL = S.make_dL_dpixels(W,H)
oc=B.Camera(); cc=cam.to_c(); C.memmove(C.byref(oc),C.byref(cc),C.sizeof(oc))
out = orc.gs_render(sc, oc, dL, threads=8, tile_stride=16, tap=True, tap_ppt=2)
tr = out['tap']
wid = np.asarray(tr.warp_id); it = np.asarray(tr.iteration)
tile = wid // 4; w = wid % 4
print("records", len(wid), "unique tiles", len(np.unique(tile)))
# per tile: bmax ~ max iteration+1 over its records (approx)
tot_persist = 0; tot_batch = 0; tot_work = 0
for t in np.unique(tile):
    m = tile == t
    its = it[m]; ws = w[m]
    top = its.max() + 1
    batch = (top - 1 - its) // 256
    nb = batch.max() + 1
    cnt = np.zeros((nb, 4))
    np.add.at(cnt, (batch, ws), 1)
    tot_work += cnt.sum()
    tot_persist += 4 * cnt.sum(axis=0).max()          # CTA time if warps never sync
    tot_batch += 4 * cnt.max(axis=1).sum()            # CTA time with a barrier per batch
print("useful warp-walks", tot_work)
print("slots with per-batch barriers", tot_batch, "efficiency %.3f" % (tot_work / tot_batch))
print("slots with no barriers (persistent imbalance only)", tot_persist, "efficiency %.3f" % (tot_work / tot_persist))
