# multi-rank factorization checks on one GPU (ranks share cuda:0 over gloo):
#   bash tools/dist_run.sh "world N form dtop transport" ...
for cfg in "$@"; do
  set -- $cfg
  PS_DIST_BACKEND=gloo PS_DIST_SAME_DEVICE=1 PS_DIST_TOP=$4 PS_DIST_TRANSPORT=$5 timeout 300 \
    python -m torch.distributed.run --nnodes=1 --nproc-per-node=$1 --master-addr 127.0.0.1 \
    --master-port 29650 tools/dist_check.py $2 $3 2>&1 | grep -v "W1017\|Warn\|OMP\|\*\*\*\*" | tail -40
done
