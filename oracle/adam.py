"""TEST INFRASTRUCTURE ONLY -- numpy restatement of the per-attribute Adam step (csrc/optim.cu).

SPEC.md:430 (mapping_round): one Adam step per attribute group with lr position 1.6e-4, rotation
1e-3, log-scale 5e-3, opacity-logit 5e-2, colour 2.5e-3, feature 2.5e-3; standard bias-corrected
Adam (beta1 0.9, beta2 0.999, eps 1e-8); SH bands above DC at colour lr / 20.  Parameters in the
reference layouts (rotation stored x,y,z,w), gradients as lego::MapGradients (rotation w,x,y,z,
feature [d][N], renderer.hpp:59-68).  Evaluated in float32 with the kernel's operation order."""
from __future__ import annotations

import numpy as np

DEFAULT = dict(lr_position=1.6e-4, lr_rotation=1e-3, lr_log_scale=5e-3, lr_opacity=5e-2, lr_color=2.5e-3,
               lr_sh_rest=2.5e-3 / 20.0, lr_feature=2.5e-3, beta1=0.9, beta2=0.999, eps=1e-8)


class AdamOracle:
    def __init__(self, scene, **cfg):
        self.c = dict(DEFAULT, **cfg)
        self.p = {k: np.array(v, np.float32, copy=True) for k, v in scene.items()}
        self.m = {k: np.zeros_like(v) for k, v in self.p.items()}
        self.v = {k: np.zeros_like(v) for k, v in self.p.items()}
        self.t = 0

    def _upd(self, key, g, lr, sl=slice(None)):
        c = self.c
        f = np.float32
        b1, b2, eps = f(c["beta1"]), f(c["beta2"]), f(c["eps"])
        c1 = f(1.0 / (1.0 - c["beta1"] ** self.t))
        c2 = f(1.0 / (1.0 - c["beta2"] ** self.t))
        g = np.asarray(g, np.float32)
        m = self.m[key][sl]
        v = self.v[key][sl]
        m = b1 * m + (f(1) - b1) * g
        v = b2 * v + (f(1) - b2) * g * g
        self.m[key][sl] = m
        self.v[key][sl] = v
        self.p[key][sl] = self.p[key][sl] - f(lr) * (m * c1) / (np.sqrt(v * c2) + eps)

    def step(self, grads):
        self.t += 1
        c = self.c
        self._upd("pos", grads["position"], c["lr_position"])
        g = np.asarray(grads["rotation"], np.float32)
        self._upd("rot", g[:, [1, 2, 3, 0]], c["lr_rotation"])  # w,x,y,z -> stored x,y,z,w
        self._upd("log_s", grads["log_scale"], c["lr_log_scale"])
        self._upd("opac", grads["opacity_logit"], c["lr_opacity"])
        gs = np.asarray(grads["sh"], np.float32)
        self._upd("sh", gs[:, :1, :], c["lr_color"], (slice(None), slice(0, 1), slice(None)))
        if gs.shape[1] > 1:
            self._upd("sh", gs[:, 1:, :], c["lr_sh_rest"], (slice(None), slice(1, None), slice(None)))
        if self.p["feat"].size:
            self._upd("feat", grads["feature"], c["lr_feature"])
        return self.p
