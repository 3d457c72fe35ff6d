#!/bin/bash
# A/B of the in-tree liblpmoe.so against the library built from another git revision.
#
#   tools/lib_ab.sh build REV            # here (CPU): builds REV in a temporary worktree and copies
#                                        #   its library to paper_2510_08055_b200/_lib/liblpmoe_ab.so
#   tools/lib_ab.sh run "T1 T2" REPS [bench.py args]   # on the GPU box: interleaved bench lines,
#                                        #   "new" = in-tree library, "old" = liblpmoe_ab.so (LPMOE_LIB)
#
# (How the round-2 A/Bs of the decode ring, the tiny ring and the router were run; their outputs are
# under profiles/r02/probe/.)
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
AB=$ROOT/paper_2510_08055_b200/_lib/liblpmoe_ab.so
case "$1" in
  build)
    WT=$(mktemp -d /tmp/lpmoe_ab.XXXX)
    git -C "$ROOT" worktree add --detach "$WT" "$2" >/dev/null
    (cd "$WT" && python -m paper_2510_08055_b200.build >/dev/null)
    cp "$WT/paper_2510_08055_b200/_lib/liblpmoe.so" "$AB"
    git -C "$ROOT" worktree remove --force "$WT"
    echo "built $2 -> $AB"
    ;;
  run)
    Ts=$2; R=$3; shift 3
    for rep in $(seq "$R"); do
      for T in $Ts; do
        timeout 300 python "$ROOT/bench.py" --tokens "$T" --steps 30 --no-cpu-baseline "$@" 2>/dev/null | sed "s/^/new /"
        LPMOE_LIB=$AB timeout 300 python "$ROOT/bench.py" --tokens "$T" --steps 30 --no-cpu-baseline "$@" 2>/dev/null | sed "s/^/old /"
      done
    done
    ;;
  *) echo "usage: $0 build REV | run \"T...\" REPS [bench args]"; exit 2 ;;
esac
