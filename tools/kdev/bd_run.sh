cd $GRAFT_REPO_ROOT
for i in 1 2; do
for W in homo hetero hetero_bits; do
X=""; [ $W = hetero_bits ] && X=1
echo "$W direct"; QD_WBITS=$X QD_W=${W%_bits} python tools/quick_d.py 2

done; done
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
