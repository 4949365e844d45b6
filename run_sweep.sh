#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "mailbox or tail" 2>&1 | tail -15
MGRX_ARNOLDI_SELFXCHG=1 timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-variant 2>&1 | tail -1 | cut -c1-200
