"""Training-side driver (§4.3, hyper-parameters P:1217): one
optimisation step per (t, camera) frame — the paper trains with batch size 1 — made only of C-ABI calls:

    fgs_deform -> fgs_render -> fgs_l1_loss (+ fgs_tv_loss) -> fgs_render_backward -> fgs_deform_backward
    -> fgs_adam_step on every parameter tensor

Python here only sequences the calls and owns the buffers (gradients, Adam moments, scratch); every
arithmetic step runs in libfgs.so.  Not the paper's full schedule (no warm-up switch, densification or
learning-rate decay): the minimal loop that exercises the backward and the optimiser end to end.
"""
from __future__ import annotations

from . import fgs

GAUSSIAN_KEYS = ("means", "log_scales", "quats", "opacity_logits", "sh")


class Trainer:
    def __init__(self, ds, lr_gaussians=1.6e-3, lr_field=1.6e-3, lr_mlp=1.6e-4, tv_weight=0.0):
        import torch
        self.ds = ds
        self.lr = {"g": lr_gaussians, "f": lr_field, "m": lr_mlp}
        self.tv_weight = tv_weight
        W, H = ds.scene.cameras[0].width, ds.scene.cameras[0].height
        dev = ds.device
        self.outs, _ = ds.alloc_deformed(1)
        self.img = torch.empty((3, H, W), device=dev)
        self.dimg = torch.empty_like(self.img)
        self.ws = ds.alloc_workspace(1)
        self.part = torch.empty(fgs.FGS_LOSS_PARTIALS, dtype=torch.float64, device=dev)
        self.l1 = torch.empty(1, device=dev)
        self.tv = torch.zeros(1, device=dev)
        self.dg, self.gt = ds.alloc_gaussian_grads()        # splat backward: dL/dG' (deformed)
        self.dc, self.ct = ds.alloc_gaussian_grads()        # canonical dL/dG out of the deformation backward
        self.df, self.ft = ds.alloc_field_grads()
        self.rs = torch.empty(fgs.fgs_render_backward_scratch_bytes(ds.n), dtype=torch.uint8, device=dev)
        self.dsb = torch.empty(fgs.fgs_deform_backward_scratch_bytes(ds.field, ds.mlp), dtype=torch.uint8, device=dev)
        # (param tensor, grad tensor, lr group) of every trainable tensor; Adam moments per tensor
        self.params = []
        # SH / logits are deformed only with the P:1232 decoders; otherwise the splat gradient is theirs
        canon_keys = {"means", "log_scales", "quats"} | ({"sh"} if ds.has_c else set()) \
            | ({"opacity_logits"} if ds.has_a else set())
        for k in GAUSSIAN_KEYS:
            grad = self.ct[k] if k in canon_keys else self.gt[k]
            self.params.append((getattr(ds, k), grad, "g"))
        for l, ps in enumerate(ds.planes):
            for p, P in enumerate(ps):
                self.params.append((P, self.ft[f"plane{l}_{p}"], "f"))
        for k in ("w_d", "b_d", "w_x", "b_x", "w_r", "b_r", "w_s", "b_s", "w_c", "b_c", "w_a", "b_a"):
            if k in self.ft:
                self.params.append((ds.mlp_t[k], self.ft[k], "m"))
        self.m = [torch.zeros_like(p) for p, _, _ in self.params]
        self.v = [torch.zeros_like(p) for p, _, _ in self.params]
        self.t = 0

    def step(self, frame, target):
        """One optimisation step on frame `frame` against the device image `target`; returns the device
        tensors (L1, w L_tv) of the step's forward (read them after the stream synchronises)."""
        ds = self.ds
        t = ds.times[frame]
        fgs.fgs_deform(ds.g, ds.field, ds.mlp, t, self.outs[0])
        fgs.fgs_render(ds.cams[frame], self.outs[0], self.img, self.ws)
        fgs.fgs_l1_loss(self.img, target, self.dimg, self.part, self.l1)
        fgs.fgs_render_backward(ds.cams[frame], self.outs[0], self.img, self.dimg, self.ws, self.rs, self.dg)
        for v in self.ft.values():
            v.zero_()                                     # field gradients of this step only (memset)
        if self.tv_weight:
            fgs.fgs_tv_loss(ds.field, self.tv_weight, self.df, self.part, self.tv)
        fgs.fgs_deform_backward(ds.g, ds.field, ds.mlp, t, self.dg, self.dc, self.df, self.dsb)
        self.t += 1
        for (p, g, grp), m, v in zip(self.params, self.m, self.v):
            fgs.fgs_adam_step(p, g, m, v, self.lr[grp], self.t)
        return self.l1, self.tv
