import sys, time; sys.path.insert(0,'/root/repo')
import numpy as np
from tools.quick_perf import synth_rom
from paper_2411_12690_b200 import configs
from paper_2411_12690_b200.api import GpuGlobalStage, ArrayLayout, IterOptions
cfg = configs.get(3)
g = GpuGlobalStage(0)
g.set_roms(synth_rom(cfg, 0))
for i in range(3):
    t = time.perf_counter(); g.set_layout(ArrayLayout(cfg.rows, cfg.cols, None, cfg.delta_t(), cfg.p, cfg.h)); t1 = time.perf_counter()
    g.set_bc("bottom_pin_321"); t2 = time.perf_counter()
    print(f"set_layout {t1-t:.3f}s set_bc {t2-t1:.3f}s", flush=True)
