#!/bin/bash
# quick GPU check: parity tests + timing
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -1
timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import numpy as np
from paper_1806_03461_b200 import tfhe
K=tfhe.KeySet(seed=42); e=tfhe.Engine(K)
lin=K.encrypt(np.random.default_rng(5).integers(0,2,512).astype(np.uint8), seed=9, stream=4)
e.debug_bootstrap_wo_ks(lin); print('fft margin over 512 bootstraps:', e.debug_fft_margin())
"
timeout 300 python scripts/gpu_timing.py 2>&1 | tail -2
