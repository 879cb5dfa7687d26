import sys, time
sys.path.insert(0, "/root/repo")
import torch
from paper_2306_07191_b200 import BvhBackend, NifBackend, build_model
from paper_2306_07191_b200.nif import NifConfig
from paper_2306_07191_b200.pipeline import render_dev, sample_pass_dev, shadow_rays_dev
from paper_2306_07191_b200.synthetic import c2
torch.cuda.set_device(0)
for (w, h) in ((1920, 1080), (3840, 2160)):
    scene = c2(w, h)
    model = build_model(NifConfig(seed=0), scene)
    nb, bb = NifBackend(model), BvhBackend()
    def tm(fn, reps=3):
        fn(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(reps): fn()
        e1.record(); e1.synchronize()
        return e0.elapsed_time(e1) / reps
    data = sample_pass_dev(scene, scene.camera, 0, scene.seed)
    cast, o, d, t = shadow_rays_dev(data)
    print(w, h, "sample pass", tm(lambda: sample_pass_dev(scene, scene.camera, 0, scene.seed)),
          "cast+compact", tm(lambda: shadow_rays_dev(data)),
          "nif occ_dev", tm(lambda: nb.occluded_dev(scene, o, d, t)),
          "bvh occ_dev", tm(lambda: bb.occluded_dev(scene, o, d, t)),
          "render nif", tm(lambda: render_dev(scene, nb, spp=1)),
          "render bvh", tm(lambda: render_dev(scene, bb, spp=1)))
