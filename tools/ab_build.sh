#!/bin/bash
# Builds the committed HEAD's libspx.so into ab_libs/libspx_head.so (git worktree in /tmp), so a
# gpurun call can A/B the working tree against HEAD on one box (SPX_LIB=ab_libs/libspx_head.so).
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
WT=/tmp/spx_head_wt
rm -rf $WT; git -C $ROOT worktree prune
git -C $ROOT worktree add -f --detach $WT ${1:-HEAD} > /dev/null
make -s -j16 -C $WT/paper_2603_06664_b200/csrc > /dev/null
mkdir -p $ROOT/ab_libs
cp $WT/paper_2603_06664_b200/libspx.so $ROOT/ab_libs/libspx_head.so
git -C $ROOT worktree remove --force $WT
echo "ab_libs/libspx_head.so <- $(git -C $ROOT rev-parse --short ${1:-HEAD})"
