# Build libchfilter.so from git ref $1 into ab_alt/ (for scripts/ab_lib.sh).
# The alt library is stamped with the current ABI version (A/B timing only:
# bench.py never reads an ABI struct whose layout changed).
set -e
REF=${1:-HEAD}
ABI=$(grep -o "define CH_ABI_VERSION [0-9]*" include/chfilter.h | awk '{print $3}')
rm -rf /tmp/alt_wt && git worktree add -f /tmp/alt_wt $REF >/dev/null 2>&1 || { git worktree prune; git worktree add -f /tmp/alt_wt $REF; }
sed -i "s/define CH_ABI_VERSION [0-9]*/define CH_ABI_VERSION $ABI/" /tmp/alt_wt/include/chfilter.h
(cd /tmp/alt_wt && python -c "import paper_2303_10581_b200.build as b; b.build(force=True)")
mkdir -p ab_alt && cp /tmp/alt_wt/paper_2303_10581_b200/libchfilter.so ab_alt/
git worktree remove --force /tmp/alt_wt
echo "built ab_alt/libchfilter.so from $REF (ABI stamped $ABI)"
