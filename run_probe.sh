#!/bin/bash
for f in 6; do MGRX_GS_FLIGHT=$f TAG=flight$f python tools/probe_gs.py; done > gpurun_out/probe_flight.log 2>&1
MGRX_GS_FLIGHT=16 TAG=flight16 python tools/probe_gs.py >> gpurun_out/probe_flight.log 2>&1
timeout 600 python -m pytest tests -q -m gpu -x -k "bit_exact or solve_parity or apply" >> gpurun_out/probe_flight.log 2>&1
echo done
