#!/bin/bash
# session 4, one call: variant timings + parity of the L2 plane variants (scripts/gpu_r2s4a.sh), then the
# evidence at the bench defaults (scripts/gpu_r2s4_final.sh: bench line, smoke, ncu launch list, --set full)
bash scripts/gpu_r2s4a.sh
bash scripts/gpu_r2s4_final.sh r02s4f
