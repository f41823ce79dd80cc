#!/bin/bash
# build libprism.so of a git ref (or the working tree: "wt") into ab/libprism_<name>.so for same-box A/B runs
# usage: tools/ab_build.sh <name> <ref|wt>
set -e
name=$1; ref=$2
mkdir -p /root/repo/ab
if [ "$ref" = "wt" ]; then
  python -c "from paper_2605_08581_b200 import build as B; B.build(force=True, verbose=False)"
  cp paper_2605_08581_b200/libprism.so ab/libprism_$name.so
else
  rm -rf /tmp/ab_$name; git worktree add -f /tmp/ab_$name $ref >/dev/null 2>&1
  (cd /tmp/ab_$name && python -c "from paper_2605_08581_b200 import build as B; B.build(force=True, verbose=False)")
  cp /tmp/ab_$name/paper_2605_08581_b200/libprism.so ab/libprism_$name.so
  git worktree remove --force /tmp/ab_$name
fi
ls -la ab/libprism_$name.so
