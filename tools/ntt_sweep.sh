#!/bin/bash
# NTT launch timing across chunk sizes (dev tool)
for c in 128 256 512 1024 0; do echo -n "chunk=$c "; HEAR_B200_NTT_CHUNK=$c python tools/ntt_probe.py | python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read().strip()); print(d['launch_us'], d['butterflies_per_s'])"; done
