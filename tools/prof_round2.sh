python tools/step_profile.py 1d-w64 full 64 > gpurun_out/sp.log 2>&1 || exit 1
grep demangled tools/prof_round.sh | bash
ls gpurun_out
