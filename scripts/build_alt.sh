# Build libchfilter.so from git ref $1 into ab_alt/ (for scripts/ab_lib.sh)
set -e
REF=${1:-HEAD}
rm -rf /tmp/alt_wt && git worktree add -f /tmp/alt_wt $REF >/dev/null 2>&1 || { git worktree prune; git worktree add -f /tmp/alt_wt $REF; }
(cd /tmp/alt_wt && python -c "import paper_2303_10581_b200.build as b; b.build(force=True)")
mkdir -p ab_alt && cp /tmp/alt_wt/paper_2303_10581_b200/libchfilter.so ab_alt/
git worktree remove --force /tmp/alt_wt
echo "built ab_alt/libchfilter.so from $REF"
