"""Hand-built tiny inputs for closed-form pins (test helper; no method arithmetic)."""
import dataclasses

import numpy as np

import scenegen


def mini(points, normals, vpl_pos, vpl_nrm, vpl_I, views=None, rho=None, spec=None, expo=None,
         sph=(), box=(), rect=(), tri=(), clamp_dist=1e-3, shadow_eps=1e-6, diag=1.0, tree=None, **cfg_over):
    P = np.atleast_2d(np.asarray(points, np.float64))
    N = np.atleast_2d(np.asarray(normals, np.float64))
    m = P.shape[0]
    V = N if views is None else np.atleast_2d(np.asarray(views, np.float64))
    R = np.ones((m, 3)) if rho is None else np.atleast_2d(np.asarray(rho, np.float64))
    S = np.zeros(m) if spec is None else np.asarray(spec, np.float64).reshape(m)
    E = np.ones(m, np.int32) if expo is None else np.asarray(expo, np.int32).reshape(m)
    f32 = np.float32
    g = dict(pixel=np.arange(m, dtype=np.int32), px=P[:, 0].astype(f32), py=P[:, 1].astype(f32), pz=P[:, 2].astype(f32),
             nx=N[:, 0].astype(f32), ny=N[:, 1].astype(f32), nz=N[:, 2].astype(f32),
             vx=V[:, 0].astype(f32), vy=V[:, 1].astype(f32), vz=V[:, 2].astype(f32),
             rho_r=R[:, 0].astype(f32), rho_g=R[:, 1].astype(f32), rho_b=R[:, 2].astype(f32),
             spec=S.astype(f32), exponent=E)
    LP = np.atleast_2d(np.asarray(vpl_pos, np.float64))
    LN = np.atleast_2d(np.asarray(vpl_nrm, np.float64))
    LI = np.atleast_2d(np.asarray(vpl_I, np.float64))
    v = dict(px=LP[:, 0].astype(f32), py=LP[:, 1].astype(f32), pz=LP[:, 2].astype(f32),
             nx=LN[:, 0].astype(f32), ny=LN[:, 1].astype(f32), nz=LN[:, 2].astype(f32),
             ir=LI[:, 0].astype(f32), ig=LI[:, 1].astype(f32), ib=LI[:, 2].astype(f32))
    if tree is None:
        tree = scenegen._light_tree(v, LP.shape[0])   # cut = all leaves
    prims = dict(sph=np.asarray(sph, f32).reshape(-1, 4), box=np.asarray(box, f32).reshape(-1, 6),
                 rect=np.asarray(rect, f32).reshape(-1, 12), tri=np.asarray(tri, f32).reshape(-1, 9))
    cfg = dataclasses.replace(scenegen.PRESETS["c1"], width=m, height=1, n_vpls=LP.shape[0], **cfg_over)
    return scenegen.Inputs(cfg=cfg, scene=None, width=m, height=1, gbuf=g, vpls=v, tree=tree, prims=prims,
                           diag=diag, clamp_dist=clamp_dist, shadow_eps=shadow_eps, tau=cfg.tau)


def rect_prim(p0, e1, e2):
    p0, e1, e2 = (np.asarray(a, np.float64) for a in (p0, e1, e2))
    return np.concatenate([p0, e1, e2, np.cross(e1, e2)])
