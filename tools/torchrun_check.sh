# the driver's scaling launch (torchrun, one rank per GPU) at N=1: default config, c4 bands, c5 batch shard, reference arm
out=gpurun_out/torchrun
mkdir -p $out
tr="python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517"
timeout 600 $tr bench.py --gpus 1 --steps 5 --warmup 3 > $out/default.log 2>&1; echo "rc=$?" >> $out/default.log
timeout 600 $tr bench.py --gpus 1 --config c4 --steps 3 --warmup 3 > $out/c4.log 2>&1; echo "rc=$?" >> $out/c4.log
timeout 900 $tr bench.py --gpus 1 --config c5 --steps 3 --warmup 3 > $out/c5.log 2>&1; echo "rc=$?" >> $out/c5.log
timeout 600 $tr bench.py --impl reference --gpus 1 --steps 3 --warmup 3 > $out/reference.log 2>&1; echo "rc=$?" >> $out/reference.log
