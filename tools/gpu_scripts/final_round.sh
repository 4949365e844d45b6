#!/bin/bash
# End-of-round evidence: launch lists (cfg2/3/4) and step timeline, then the
# round check (GPU suite, smoke, cfg2 bench + reference arm, cfg3-5 benches).
bash tools/gpu_scripts/launch_lists.sh
bash tools/gpu_scripts/round_check.sh
