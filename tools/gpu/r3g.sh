#!/bin/bash
out=gpurun_out/r3g
mkdir -p $out
export TSV_NO_BUILD=1 TSV_SYM_STAGGER_NS=0
for gr in 296 222 148 74; do for ab in 0 3 4 6; do echo "grid $gr ablate $ab: $(TSV_SYM_GRID=$gr TSV_SYM_ABLATE=$ab python tools/k1_only.py 3 20)"; done; done 2>&1 | tee $out/grid.log
