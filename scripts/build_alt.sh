# Build libchfilter.so from git ref $1 into build/alt/ (for scripts/ab_lib.sh)
set -e
REF=${1:-HEAD}
rm -rf /tmp/alt_wt && git worktree add -f /tmp/alt_wt $REF >/dev/null 2>&1 || { git worktree prune; git worktree add -f /tmp/alt_wt $REF; }
(cd /tmp/alt_wt && python -c "import paper_2303_10581_b200.build as b; b.build(force=True)")
mkdir -p build/alt && cp /tmp/alt_wt/paper_2303_10581_b200/libchfilter.so build/alt/
git worktree remove --force /tmp/alt_wt
echo "built build/alt/libchfilter.so from $REF"
