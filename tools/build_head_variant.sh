# Build the committed (HEAD) version of one source into _lib/head for an A/B
# against the working tree:  bash tools/build_head_variant.sh csrc/staged.cu
set -e
f=paper_1905_03748_b200/$1
cp $f /tmp/_ab_work.cu
git show HEAD:$f > $f
python -c "from paper_1905_03748_b200 import build as b; print(b.build(force=True, out_dir='paper_1905_03748_b200/_lib/head'))" || true
cp /tmp/_ab_work.cu $f
touch $f
