#!/bin/bash
# Build build/ab/A.so from HEAD and build/ab/B.so from the working tree (dev aid for scripts/ab.sh)
set -e
cd "$(dirname "$0")/.."
mkdir -p build/ab
python -c "from paper_2603_16435_b200 import build; build.build()" && cp paper_2603_16435_b200/lib/libvqkv_b200.so build/ab/B.so
git stash -q
trap 'git stash pop -q' EXIT
touch paper_2603_16435_b200/csrc/*.cu
python -c "from paper_2603_16435_b200 import build; build.build()" && cp paper_2603_16435_b200/lib/libvqkv_b200.so build/ab/A.so
git stash pop -q; trap - EXIT
touch paper_2603_16435_b200/csrc/*.cu
python -c "from paper_2603_16435_b200 import build; build.build()"
cmp -s build/ab/B.so paper_2603_16435_b200/lib/libvqkv_b200.so || cp paper_2603_16435_b200/lib/libvqkv_b200.so build/ab/B.so
echo "A=HEAD B=worktree built"
