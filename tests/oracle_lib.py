"""Test-side loader for the CPU parity oracles (oracle/liboracle*.so, oracle/_ref/libsplat_ref*.so).

TEST INFRASTRUCTURE: imported only by tests/, __graft_entry__.smoke() and bench.py's CPU legs.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

from paper_2411_12788_b200.capi import AdamConfig, Camera, Gaussians, RasterConfig

ROOT = Path(__file__).resolve().parents[1]
ORACLE_DIR = ROOT / "oracle"
LIBS = {
    ("oracle", "B"): ORACLE_DIR / "liboracle.so",
    ("oracle", "A"): ORACLE_DIR / "liboracle_libm.so",
    ("ref", "B"): ORACLE_DIR / "_ref" / "libsplat_ref.so",
    ("ref", "A"): ORACLE_DIR / "_ref" / "libsplat_ref_libm.so",
}

fp = C.POINTER(C.c_float)
ip = C.POINTER(C.c_int32)
u8p = C.POINTER(C.c_uint8)
i64p = C.POINTER(C.c_int64)


def build_oracle() -> None:
    """(Re)build the oracle libraries (and oracle/_ref when /root/reference is present)."""
    subprocess.run(["make", "-s", "-C", str(ORACLE_DIR), "all"], check=True)


def available(kind: str, mode: str = "B") -> bool:
    return LIBS[(kind, mode)].exists()


def _ptr(a, t=fp):
    if a is None:
        return t()
    return a.ctypes.data_as(t)


class GaussiansView:
    """Keeps numpy arrays alive while a Gaussians struct points at them."""

    def __init__(self, s):
        self.arrays = [np.ascontiguousarray(x, dtype=np.float32) for x in
                       (s.centers, s.log_scales, s.rotations, s.opacity_logits, s.sh)]
        c, ls, r, o, sh = self.arrays
        self.struct = Gaussians(_ptr(c), _ptr(ls), _ptr(r), _ptr(o), _ptr(sh), s.n,
                                s.active_sh_degree)


class OracleLib:
    """One oracle implementation (C restatement or the reference build) in one exp mode."""

    def __init__(self, kind: str = "oracle", mode: str = "B"):
        self.kind, self.mode = kind, mode
        path = LIBS[(kind, mode)]
        if not path.exists():
            build_oracle()
        self.lib = C.CDLL(str(path))
        p = kind + "_"
        self.p = p
        L = self.lib
        G, CAM, CFG = C.POINTER(Gaussians), C.POINTER(Camera), C.POINTER(RasterConfig)
        getattr(L, p + "last_error").restype = C.c_char_p
        getattr(L, p + "project").argtypes = [G, CAM, CFG, u8p, ip, ip, ip, ip, fp, fp, fp, fp, fp]
        getattr(L, p + "tiles").argtypes = [G, CAM, CFG, u8p, i64p, ip, ip, C.c_int64]
        getattr(L, p + "render").argtypes = [G, CAM, CFG, u8p, fp, fp, fp, fp, fp, ip, fp, fp, ip, i64p]
        getattr(L, p + "render_backward").argtypes = [G, CAM, CFG, fp, u8p, fp, fp, fp, fp, fp, fp, fp, ip]
        getattr(L, p + "l1_loss").argtypes = [fp, fp, C.c_int64, fp]
        getattr(L, p + "l1_loss").restype = C.c_float
        getattr(L, p + "lr_at").argtypes = [C.POINTER(AdamConfig), C.c_int32]
        getattr(L, p + "lr_at").restype = C.c_double
        getattr(L, p + "exp").argtypes = [C.c_float]
        getattr(L, p + "exp").restype = C.c_float
        for fn in ("project", "tiles", "render", "render_backward"):
            getattr(L, p + fn).restype = C.c_int
        getattr(L, p + "third_neighbor_distances").argtypes = [fp, C.c_int32, C.c_float, fp]
        getattr(L, p + "ssim").argtypes = [fp, fp, C.c_int, C.c_int, C.c_int, fp]
        getattr(L, p + "ssim").restype = C.c_float
        getattr(L, p + "photometric_loss").argtypes = [fp, fp, C.c_int, C.c_int, C.c_int, C.c_float, fp]
        getattr(L, p + "photometric_loss").restype = C.c_float
        if kind == "oracle":
            getattr(L, p + "adam_step").argtypes = [fp, fp, fp, fp, fp, C.c_int32, fp, fp, fp, fp, fp, fp, fp,
                                          C.POINTER(AdamConfig), ip, C.c_uint32]
            getattr(L, p + "unproject").argtypes = [CAM, ip, fp, fp, C.c_int, C.c_float, C.c_int64, C.c_int32,
                                          C.c_int64, fp, ip, C.c_int64, i64p]
            dp = C.POINTER(C.c_double)
            getattr(L, p + "quantile_threshold").argtypes = [fp, u8p, C.c_int32, C.c_double, fp, ip]
            getattr(L, p + "quantile_threshold_f64").argtypes = [dp, u8p, C.c_int32, C.c_double, dp, ip]
            getattr(L, p + "visibility_mask").argtypes = [fp, C.c_int32, C.c_double, u8p]
            getattr(L, p + "identify_critical").argtypes = [G, fp, i64p, dp, C.c_int, C.c_double, dp, u8p, ip]
            getattr(L, p + "aggressive_clone").argtypes = [fp, fp, fp, fp, fp, C.c_int32, C.c_int64, u8p, ip, ip]
            getattr(L, p + "importance_prune").argtypes = [dp, C.c_int32, C.c_double, ip, ip]
            getattr(L, p + "reinit_gaussians").argtypes = [fp, fp, C.c_int32, C.c_float, fp, fp, fp, fp, fp]
        else:
            getattr(L, p + "adam_steps").argtypes = [fp, fp, fp, fp, fp, C.c_int32, fp, fp, fp, fp, fp,
                                           C.POINTER(AdamConfig), C.c_int32]
            getattr(L, p + "depth_reinitialize").argtypes = [G, CAM, CFG, fp, C.c_int32, C.c_uint32, fp, ip]
            dp = C.POINTER(C.c_double)
            getattr(L, p + "render_backward_f64").argtypes = [G, CAM, CFG, fp, u8p, fp, dp, dp, dp, dp, dp]
            getattr(L, p + "global_importance").argtypes = [G, CAM, C.c_int32, CFG, C.POINTER(C.c_double), ip]
            getattr(L, p + "random_scores").argtypes = [C.c_uint32, C.c_int32, dp]
            getattr(L, p + "fisher_yates").argtypes = [C.c_uint32, C.c_int32, C.c_int32, ip]
            getattr(L, p + "depth_reinitialize_views").argtypes = [G, CAM, C.c_int32, CFG, fp, C.c_int32, C.c_uint32,
                                                                   fp, fp, fp, fp, fp, ip]
            getattr(L, p + "identify_critical_views").argtypes = [G, CAM, C.c_int32, CFG, C.c_int, C.c_double,
                                                                  C.c_uint32, u8p, u8p, ip]
            getattr(L, p + "aggressive_clone_apply").argtypes = [G, u8p, fp, fp, fp, fp, fp, C.c_int64, ip, ip]
            getattr(L, p + "build_masks").argtypes = [G, CAM, C.c_int32, CFG, C.c_double, u8p]
            getattr(L, p + "importance_prune_set").argtypes = [G, dp, C.c_double, ip, ip]

        dp = C.POINTER(C.c_double)
        getattr(L, p + "rng_normal_f32").argtypes = [C.c_uint32, C.c_int32, fp]
        getattr(L, p + "rng_mixed_64").argtypes = [C.c_uint64, C.c_int32, ip, ip, ip, dp]
        if kind == "oracle":
            getattr(L, p + "adam_step_range").argtypes = [fp, fp, fp, fp, C.c_int32, C.c_int64, C.c_int64,
                                                          C.POINTER(AdamConfig), C.c_int32, C.c_uint32]
            getattr(L, p + "quat_normalize").argtypes = [fp, C.c_int32]
            getattr(L, p + "rng_uniform_f64_32").argtypes = [C.c_uint32, C.c_int32, dp]
            getattr(L, p + "rng_fisher_yates").argtypes = [C.c_uint32, C.c_int32, C.c_int32, ip]
            getattr(L, p + "importance_sample").argtypes = [dp, C.c_int32, C.c_int32, C.c_uint64, ip, ip]
            getattr(L, p + "vanilla_clone_split").argtypes = [G, fp, ip, C.c_float, C.c_float, C.c_float, C.c_uint32,
                                                              fp, fp, fp, fp, fp, C.c_int64, ip, ip, ip, ip]
        else:
            getattr(L, p + "importance_sample_set").argtypes = [G, dp, C.c_int32, C.c_uint64, ip, ip]
            getattr(L, p + "vanilla_clone_split_apply").argtypes = [G, fp, ip, C.c_float, C.c_float, C.c_float,
                                                                    C.c_uint32, fp, fp, fp, fp, fp, C.c_int64, ip, ip,
                                                                    ip, ip]

    def fn(self, name):
        return getattr(self.lib, self.p + name)

    def check(self, rc):
        if rc != 0:
            msg = self.fn("last_error")().decode()
            raise RuntimeError(f"{self.p}: status {rc}: {msg}")

    def exp(self, x: float) -> float:
        return self.fn("exp")(x)

    # ---- wrappers returning numpy --------------------------------------------------------
    def project(self, s, cam, cfg=None, mask=None):
        cfg = cfg or RasterConfig()
        gv = GaussiansView(s)
        n = s.n
        out = dict(order=np.zeros(max(n, 1), np.int32), rect=np.zeros((max(n, 1), 4), np.int32),
                   radius=np.zeros(max(n, 1), np.int32), depth=np.zeros(max(n, 1), np.float32),
                   mean2d=np.zeros((max(n, 1), 2), np.float32), conic=np.zeros((max(n, 1), 3), np.float32),
                   color=np.zeros((max(n, 1), 3), np.float32), opacity=np.zeros(max(n, 1), np.float32))
        ns = C.c_int32(0)
        m = None if mask is None else np.ascontiguousarray(mask, np.uint8)
        self.check(self.fn("project")(C.byref(gv.struct), C.byref(cam), C.byref(cfg), _ptr(m, u8p),
                                      C.byref(ns), _ptr(out["order"], ip), _ptr(out["rect"], ip),
                                      _ptr(out["radius"], ip), _ptr(out["depth"]), _ptr(out["mean2d"]),
                                      _ptr(out["conic"]), _ptr(out["color"]), _ptr(out["opacity"])))
        out = {k: v[:n] for k, v in out.items()}
        out["order"] = out["order"][: ns.value]
        out["n_survivors"] = ns.value
        return out

    def tiles(self, s, cam, cfg=None, mask=None):
        cfg = cfg or RasterConfig()
        gv = GaussiansView(s)
        tx = (cam.width + cfg.tile_size - 1) // cfg.tile_size
        ty = (cam.height + cfg.tile_size - 1) // cfg.tile_size
        ranges = np.zeros((tx * ty, 2), np.int32)
        npairs = C.c_int64(0)
        m = None if mask is None else np.ascontiguousarray(mask, np.uint8)
        self.check(self.fn("tiles")(C.byref(gv.struct), C.byref(cam), C.byref(cfg), _ptr(m, u8p),
                                    C.byref(npairs), _ptr(ranges, ip), ip(), 0))
        gauss = np.zeros(max(npairs.value, 1), np.int32)
        self.check(self.fn("tiles")(C.byref(gv.struct), C.byref(cam), C.byref(cfg), _ptr(m, u8p),
                                    C.byref(npairs), _ptr(ranges, ip), _ptr(gauss, ip), npairs.value))
        return dict(ranges=ranges, gaussian=gauss[: npairs.value], n_pairs=npairs.value,
                    tiles_x=tx, tiles_y=ty)

    def render(self, s, cam, cfg=None, mask=None, bg=(0.0, 0.0, 0.0), report=True):
        cfg = cfg or RasterConfig()
        gv = GaussiansView(s)
        h, w, n = cam.height, cam.width, s.n
        o = dict(color=np.zeros((h, w, 3), np.float32), alpha=np.zeros((h, w), np.float32),
                 depth=np.zeros((h, w), np.float32), transmittance=np.zeros((h, w), np.float32),
                 max_contributor=np.zeros((h, w), np.int32))
        r = dict(importance=np.zeros(max(n, 1), np.float32), max_weight=np.zeros(max(n, 1), np.float32),
                 max_pixel_count=np.zeros(max(n, 1), np.int32)) if report else {}
        stats = np.zeros(2, np.int64)
        bgv = np.asarray(bg, np.float32)
        m = None if mask is None else np.ascontiguousarray(mask, np.uint8)
        self.check(self.fn("render")(
            C.byref(gv.struct), C.byref(cam), C.byref(cfg), _ptr(m, u8p), _ptr(bgv),
            _ptr(o["color"]), _ptr(o["alpha"]), _ptr(o["depth"]), _ptr(o["transmittance"]),
            _ptr(o["max_contributor"], ip), _ptr(r.get("importance")), _ptr(r.get("max_weight")),
            _ptr(r.get("max_pixel_count"), ip), _ptr(stats, i64p)))
        o.update({k: v[:n] for k, v in r.items()})
        o["visits"], o["commits"] = int(stats[0]), int(stats[1])
        return o

    def render_backward(self, s, cam, d_color, cfg=None, mask=None, bg=(0.0, 0.0, 0.0)):
        cfg = cfg or RasterConfig()
        gv = GaussiansView(s)
        n = max(s.n, 1)
        g = dict(d_centers=np.zeros((n, 3), np.float32), d_log_scales=np.zeros((n, 3), np.float32),
                 d_rotations=np.zeros((n, 4), np.float32), d_opacity_logits=np.zeros(n, np.float32),
                 d_sh=np.zeros((n, 48), np.float32), grad2d_accum=np.zeros(n, np.float32),
                 grad2d_count=np.zeros(n, np.int32))
        dc = np.ascontiguousarray(d_color, np.float32)
        bgv = np.asarray(bg, np.float32)
        m = None if mask is None else np.ascontiguousarray(mask, np.uint8)
        self.check(self.fn("render_backward")(
            C.byref(gv.struct), C.byref(cam), C.byref(cfg), _ptr(dc), _ptr(m, u8p), _ptr(bgv),
            _ptr(g["d_centers"]), _ptr(g["d_log_scales"]), _ptr(g["d_rotations"]),
            _ptr(g["d_opacity_logits"]), _ptr(g["d_sh"]), _ptr(g["grad2d_accum"]),
            _ptr(g["grad2d_count"], ip)))
        return {k: v[: s.n] for k, v in g.items()}

    def render_backward_f64(self, s, cam, d_color, cfg=None, mask=None, bg=(0.0, 0.0, 0.0)):
        """Reference render_backward<double> (fp64 truth) on the float inputs."""
        cfg = cfg or RasterConfig()
        gv = GaussiansView(s)
        n = max(s.n, 1)
        g = dict(d_centers=np.zeros((n, 3)), d_log_scales=np.zeros((n, 3)), d_rotations=np.zeros((n, 4)),
                 d_opacity_logits=np.zeros(n), d_sh=np.zeros((n, 48)))
        dc = np.ascontiguousarray(d_color, np.float32)
        bgv = np.asarray(bg, np.float32)
        m = None if mask is None else np.ascontiguousarray(mask, np.uint8)
        dptr = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))
        self.check(self.fn("render_backward_f64")(
            C.byref(gv.struct), C.byref(cam), C.byref(cfg), _ptr(dc), _ptr(m, u8p), _ptr(bgv),
            dptr(g["d_centers"]), dptr(g["d_log_scales"]), dptr(g["d_rotations"]), dptr(g["d_opacity_logits"]),
            dptr(g["d_sh"])))
        return {k: v[: s.n] for k, v in g.items()}

    def l1_loss(self, a, b, want_grad=True):
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        grad = np.zeros_like(a) if want_grad else None
        loss = self.fn("l1_loss")(_ptr(a), _ptr(b), a.size, _ptr(grad))
        return float(loss), grad

    def lr_at(self, cfg, step):
        return self.fn("lr_at")(C.byref(cfg), step)

    def adam_step(self, s, grads, m, v, cfg, step, group_mask=31):
        """oracle_adam_step in place on copies; returns (set, m, v, step)."""
        s = s.copy()
        m = np.ascontiguousarray(m, np.float32).copy()
        v = np.ascontiguousarray(v, np.float32).copy()
        st = C.c_int32(step)
        gr = {k: np.ascontiguousarray(grads[k], np.float32) for k in
              ("d_centers", "d_log_scales", "d_rotations", "d_opacity_logits", "d_sh")}
        self.check(self.fn("adam_step")(
            _ptr(s.centers), _ptr(s.log_scales), _ptr(s.rotations), _ptr(s.opacity_logits), _ptr(s.sh),
            s.n, _ptr(gr["d_centers"]), _ptr(gr["d_log_scales"]), _ptr(gr["d_rotations"]),
            _ptr(gr["d_opacity_logits"]), _ptr(gr["d_sh"]), _ptr(m), _ptr(v), C.byref(cfg),
            C.byref(st), group_mask))
        return s, m, v, st.value

    def adam_steps(self, s, grads, cfg, steps):
        """ref_adam_steps: `steps` reference OptimState::step calls from zero moments."""
        s = s.copy()
        gr = {k: np.ascontiguousarray(grads[k], np.float32) for k in
              ("d_centers", "d_log_scales", "d_rotations", "d_opacity_logits", "d_sh")}
        self.check(self.fn("adam_steps")(
            _ptr(s.centers), _ptr(s.log_scales), _ptr(s.rotations), _ptr(s.opacity_logits), _ptr(s.sh),
            s.n, _ptr(gr["d_centers"]), _ptr(gr["d_log_scales"]), _ptr(gr["d_rotations"]),
            _ptr(gr["d_opacity_logits"]), _ptr(gr["d_sh"]), C.byref(cfg), steps))
        return s

    def unproject(self, cam, max_contributor, alpha, depth, rule=0, alpha_threshold=0.5,
                  view_index=0, stride=1, seed=0):
        hw = cam.width * cam.height
        pts = np.zeros((hw, 3), np.float32)
        pix = np.zeros(hw, np.int32)
        cnt = C.c_int64(0)
        mc = np.ascontiguousarray(max_contributor, np.int32)
        al = np.ascontiguousarray(alpha, np.float32)
        dp = np.ascontiguousarray(depth, np.float32)
        self.check(self.fn("unproject")(C.byref(cam), _ptr(mc, ip), _ptr(al), _ptr(dp), rule,
                                        alpha_threshold, view_index, stride, seed, _ptr(pts),
                                        _ptr(pix, ip), hw, C.byref(cnt)))
        return pts[: cnt.value], pix[: cnt.value]

    def depth_reinitialize(self, s, cam, image, sample_count, seed=0, cfg=None):
        cfg = cfg or RasterConfig()
        gv = GaussiansView(s)
        out = np.zeros((cam.width * cam.height, 3), np.float32)
        cnt = C.c_int32(0)
        img = np.ascontiguousarray(image, np.float32)
        self.check(self.fn("depth_reinitialize")(C.byref(gv.struct), C.byref(cam), C.byref(cfg),
                                                 _ptr(img), sample_count, seed, _ptr(out), C.byref(cnt)))
        return out[: cnt.value]

    def global_importance(self, s, cams, cfg=None):
        cfg = cfg or RasterConfig()
        gv = GaussiansView(s)
        arr = (Camera * len(cams))(*cams)
        acc = np.zeros(s.n, np.float64)
        cnt = np.zeros(s.n, np.int32)
        self.check(self.fn("global_importance")(C.byref(gv.struct), arr, len(cams), C.byref(cfg),
                                                acc.ctypes.data_as(C.POINTER(C.c_double)), _ptr(cnt, ip)))
        return acc, cnt

    # ---- densification / simplification -----------------------------------
    def quantile_threshold(self, values, keep_q, sel=None):
        v = np.ascontiguousarray(values)
        sel = None if sel is None else np.ascontiguousarray(sel, np.uint8)
        cnt = C.c_int32()
        if v.dtype == np.float64:
            tau = C.c_double()
            self.check(self.fn("quantile_threshold_f64")(_ptr(v, C.POINTER(C.c_double)), _ptr(sel, u8p), v.size,
                                                         keep_q, C.byref(tau), C.byref(cnt)))
        else:
            v = v.astype(np.float32)
            tau = C.c_float()
            self.check(self.fn("quantile_threshold")(_ptr(v), _ptr(sel, u8p), v.size, keep_q, C.byref(tau),
                                                     C.byref(cnt)))
        return tau.value, cnt.value

    def visibility_mask(self, importance, keep_q):
        imp = np.ascontiguousarray(importance, np.float32)
        mask = np.zeros(imp.size, np.uint8)
        self.check(self.fn("visibility_mask")(_ptr(imp), imp.size, keep_q, _ptr(mask, u8p)))
        return mask

    def view_statistics(self, s, cams, cfg=None, masks=None):
        """Per-view accumulate_importance folded into (best weight, max-count sum, fp64 summed)."""
        best = np.zeros(s.n, np.float32)
        cnt = np.zeros(s.n, np.int64)
        summed = np.zeros(s.n, np.float64)
        for k, cam in enumerate(cams):
            r = self.render(s, cam, cfg, mask=None if masks is None else masks[k])
            best = np.maximum(best, r["max_weight"])
            cnt += r["max_pixel_count"]
            summed += r["importance"].astype(np.float64)
        return best, cnt, summed

    def identify_critical(self, s, best, max_count_sum, summed, criterion, keep_q, random=None):
        gv = GaussiansView(s)
        best = np.ascontiguousarray(best, np.float32)
        mc = np.ascontiguousarray(max_count_sum, np.int64)
        sm = np.ascontiguousarray(summed, np.float64)
        rnd = None if random is None else np.ascontiguousarray(random, np.float64)
        crit = np.zeros(s.n, np.uint8)
        cnt = C.c_int32()
        dp = C.POINTER(C.c_double)
        self.check(self.fn("identify_critical")(C.byref(gv.struct), _ptr(best), _ptr(mc, i64p), _ptr(sm, dp),
                                                criterion, keep_q, _ptr(rnd, dp), _ptr(crit, u8p), C.byref(cnt)))
        return crit, cnt.value

    def aggressive_clone(self, s, critical):
        n = s.n
        cap = 2 * n
        arr = [np.zeros((cap, w), np.float32) for w in (3, 3, 4)] + [np.zeros(cap, np.float32),
                                                                     np.zeros((cap, 48), np.float32)]
        for a, src in zip(arr, (s.centers, s.log_scales, s.rotations, s.opacity_logits, s.sh)):
            a[:n] = src
        ms = np.zeros(cap, np.int32)
        n_out = C.c_int32()
        crit = np.ascontiguousarray(critical, np.uint8)
        if self.kind == "oracle":
            self.check(self.fn("aggressive_clone")(*[_ptr(a) for a in arr], n, cap, _ptr(crit, u8p), _ptr(ms, ip),
                                                   C.byref(n_out)))
        else:
            gv = GaussiansView(s)
            self.check(self.fn("aggressive_clone_apply")(C.byref(gv.struct), _ptr(crit, u8p), *[_ptr(a) for a in arr],
                                                         cap, _ptr(ms, ip), C.byref(n_out)))
        m = n_out.value
        return [a[:m] for a in arr], ms[:m]

    def importance_prune(self, importance, keep_q, s=None):
        imp = np.ascontiguousarray(importance, np.float64)
        kept = np.zeros(max(imp.size, 1), np.int32)
        nk = C.c_int32()
        dp = C.POINTER(C.c_double)
        if self.kind == "oracle":
            self.check(self.fn("importance_prune")(_ptr(imp, dp), imp.size, keep_q, _ptr(kept, ip), C.byref(nk)))
        else:
            gv = GaussiansView(s)
            self.check(self.fn("importance_prune_set")(C.byref(gv.struct), _ptr(imp, dp), keep_q, _ptr(kept, ip),
                                                       C.byref(nk)))
        return kept[: nk.value]

    # reference-only entry points
    def random_scores(self, seed, n):
        out = np.zeros(n, np.float64)
        self.check(self.fn("random_scores")(seed, n, _ptr(out, C.POINTER(C.c_double))))
        return out

    def identify_critical_views(self, s, cams, criterion, keep_q, seed=0, cfg=None, masks=None):
        gv = GaussiansView(s)
        cam_arr = (Camera * len(cams))(*cams)
        m = None if masks is None else np.ascontiguousarray(masks, np.uint8)
        crit = np.zeros(s.n, np.uint8)
        cnt = C.c_int32()
        self.check(self.fn("identify_critical_views")(C.byref(gv.struct), cam_arr, len(cams), C.byref(cfg or RasterConfig()),
                                                      criterion, keep_q, seed, _ptr(m, u8p), _ptr(crit, u8p),
                                                      C.byref(cnt)))
        return crit, cnt.value

    def build_masks(self, s, cams, keep_q, cfg=None):
        gv = GaussiansView(s)
        cam_arr = (Camera * len(cams))(*cams)
        masks = np.zeros((len(cams), s.n), np.uint8)
        self.check(self.fn("build_masks")(C.byref(gv.struct), cam_arr, len(cams), C.byref(cfg or RasterConfig()), keep_q,
                                          _ptr(masks, u8p)))
        return masks

    # ---- SSIM / photometric loss (loss.cpp:78-147) ------------------------------------------
    def ssim(self, a, b, want_grad=True):
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        h, w, ch = a.shape
        g = np.zeros_like(a) if want_grad else None
        v = self.fn("ssim")(_ptr(a), _ptr(b), w, h, ch, _ptr(g))
        return float(v), g

    def photometric_loss(self, rendered, target, lam, want_grad=True):
        a = np.ascontiguousarray(rendered, np.float32)
        b = np.ascontiguousarray(target, np.float32)
        h, w, ch = a.shape
        g = np.zeros_like(a) if want_grad else None
        v = self.fn("photometric_loss")(_ptr(a), _ptr(b), w, h, ch, lam, _ptr(g))
        return float(v), g

    # ---- depth re-initialisation tail (spatial.cpp, densify.cpp:227-251) ----------------------
    def third_neighbor_distances(self, points, min_dist=1e-7):
        p = np.ascontiguousarray(points, np.float32).reshape(-1, 3)
        out = np.zeros(max(p.shape[0], 1), np.float32)
        self.check(self.fn("third_neighbor_distances")(_ptr(p), p.shape[0], min_dist, _ptr(out)))
        return out[: p.shape[0]]

    def reinit_gaussians(self, points, colors, min_dist=1e-7):
        p = np.ascontiguousarray(points, np.float32).reshape(-1, 3)
        col = None if colors is None else np.ascontiguousarray(colors, np.float32).reshape(-1, 3)
        m = p.shape[0]
        out = [np.zeros((m, 3), np.float32), np.zeros((m, 3), np.float32), np.zeros((m, 4), np.float32),
               np.zeros(m, np.float32), np.zeros((m, 48), np.float32)]
        self.check(self.fn("reinit_gaussians")(_ptr(p), _ptr(col), m, min_dist, *[_ptr(a) for a in out]))
        return out

    def fisher_yates(self, seed, pool, take):
        out = np.zeros(max(take, 1), np.int32)
        self.check(self.fn("fisher_yates")(seed, pool, take, _ptr(out, ip)))
        return out[:take]

    def depth_reinitialize_views(self, s, cams, images, sample_count, seed=0, cfg=None):
        gv = GaussiansView(s)
        cam_arr = (Camera * len(cams))(*cams)
        imgs = np.ascontiguousarray(np.concatenate([np.asarray(i, np.float32).reshape(-1) for i in images]))
        cap = sample_count
        out = [np.zeros((cap, 3), np.float32), np.zeros((cap, 3), np.float32), np.zeros((cap, 4), np.float32),
               np.zeros(cap, np.float32), np.zeros((cap, 48), np.float32)]
        cnt = C.c_int32()
        self.check(self.fn("depth_reinitialize_views")(C.byref(gv.struct), cam_arr, len(cams), C.byref(cfg or RasterConfig()),
                                                       _ptr(imgs), sample_count, seed, *[_ptr(a) for a in out],
                                                       C.byref(cnt)))
        return [a[: cnt.value] for a in out]

    # ---- the reference's random draws and their §8f consumers ------------------------------
    def rng_normal_f32(self, seed, n):
        out = np.zeros(max(n, 1), np.float32)
        self.check(self.fn("rng_normal_f32")(seed, n, _ptr(out)))
        return out[:n]

    def rng_mixed_64(self, seed, kinds, lo, hi):
        k, l, h = (np.ascontiguousarray(a, np.int32) for a in (kinds, lo, hi))
        out = np.zeros(max(k.size, 1), np.float64)
        self.check(self.fn("rng_mixed_64")(seed, k.size, _ptr(k, ip), _ptr(l, ip), _ptr(h, ip),
                                           _ptr(out, C.POINTER(C.c_double))))
        return out[:k.size]

    def rng_uniform_f64_32(self, seed, n):
        if self.kind == "ref":
            return self.random_scores(seed, n)
        out = np.zeros(max(n, 1), np.float64)
        self.check(self.fn("rng_uniform_f64_32")(seed, n, _ptr(out, C.POINTER(C.c_double))))
        return out[:n]

    def rng_fisher_yates(self, seed, pool, take):
        out = np.zeros(max(take, 1), np.int32)
        self.check(self.fn("rng_fisher_yates" if self.kind == "oracle" else "fisher_yates")(seed, pool, take,
                                                                                              _ptr(out, ip)))
        return out[:take]

    def importance_sample(self, importance, target, seed, s=None):
        imp = np.ascontiguousarray(importance, np.float64)
        kept = np.zeros(max(imp.size, 1), np.int32)
        nk = C.c_int32()
        dp = C.POINTER(C.c_double)
        if self.kind == "oracle":
            self.check(self.fn("importance_sample")(_ptr(imp, dp), imp.size, target, seed, _ptr(kept, ip), C.byref(nk)))
        else:
            gv = GaussiansView(s)
            self.check(self.fn("importance_sample_set")(C.byref(gv.struct), _ptr(imp, dp), target, seed, _ptr(kept, ip),
                                                        C.byref(nk)))
        return kept[:nk.value]

    def vanilla_clone_split(self, s, grad2d_accum, grad2d_count, grad_threshold, scale_threshold, scene_extent, seed):
        """Returns (GaussianSet after apply_densify_plan, moment_source, n_clone, n_split)."""
        from paper_2411_12788_b200.scenes import GaussianSet
        gv = GaussiansView(s)
        acc = np.ascontiguousarray(grad2d_accum, np.float32)
        cnt = np.ascontiguousarray(grad2d_count, np.int32)
        cap = 3 * s.n + 1
        out = GaussianSet.empty(cap, s.active_sh_degree)
        ms = np.zeros(cap, np.int32)
        no, nc, ns = C.c_int32(), C.c_int32(), C.c_int32()
        name = "vanilla_clone_split" if self.kind == "oracle" else "vanilla_clone_split_apply"
        self.check(self.fn(name)(C.byref(gv.struct), _ptr(acc), _ptr(cnt, ip), grad_threshold, scale_threshold,
                                 scene_extent, seed, _ptr(out.centers), _ptr(out.log_scales), _ptr(out.rotations),
                                 _ptr(out.opacity_logits), _ptr(out.sh), cap, _ptr(ms, ip), C.byref(no), C.byref(nc),
                                 C.byref(ns)))
        m = no.value
        return out.select(np.arange(m)), ms[:m], nc.value, ns.value

    def adam_step_range(self, params, grad_shard, m, v, n, begin, count, cfg, step, group_mask):
        """In place on float32 numpy arrays (packed layout, + padding)."""
        self.check(self.fn("adam_step_range")(_ptr(params), _ptr(grad_shard), _ptr(m), _ptr(v), n, begin, count,
                                              C.byref(cfg), step, group_mask))

    def quat_normalize(self, rotations, n):
        self.check(self.fn("quat_normalize")(_ptr(rotations), n))

