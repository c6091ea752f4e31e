#!/bin/bash
# Builds a debug copy of the library with per-scenario loop-iteration counters
# (BSG_PROFILE_ITERS: result.detail = general steps, result.member_steps = windows)
# plus any extra defines ($ITER_FLAGS) into /tmp and runs tools/iterprobe.py.
set -e
exec bash tools/variant.sh "-DBSG_PROFILE_ITERS $ITER_FLAGS" tools/iterprobe.py "$@"
