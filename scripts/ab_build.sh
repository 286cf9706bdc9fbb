#!/bin/bash
# Builds libtcse.so of git revision $1 into ab/$2.so (A/B kernel timing:
# TCSE_LIBRARY=ab/$2.so python scripts/probe_perf.py ...).
set -e
rev=$1; name=$2
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=$(mktemp -d)
git -C "$root" worktree add --detach "$tmp" "$rev" >/dev/null
(cd "$tmp" && python paper_2512_13365_b200/build.py >/dev/null)
mkdir -p "$root/ab"
cp "$tmp/paper_2512_13365_b200/libtcse.so" "$root/ab/$name.so"
git -C "$root" worktree remove --force "$tmp"
echo "$root/ab/$name.so"
