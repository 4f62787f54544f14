export HG_BENCH_ONE_GPU=1
for N in 2 8; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus $N --steps 3 --warmup 3 --layers 4 --no-cpu-baseline > gpurun_out/rehearse_$N.log 2>&1
  echo "N=$N rc=$?"; tail -c 1500 gpurun_out/rehearse_$N.log
done
