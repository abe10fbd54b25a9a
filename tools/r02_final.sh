#!/bin/bash
# round-2 evidence set (1 x B200): GPU tests, smoke, the driver's bench lines, torchrun N=1
python -m pytest tests -x -q -m gpu > gpurun_out/final_pytest.txt 2>&1; echo rc=$? >> gpurun_out/final_pytest.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.txt 2>&1; echo rc=$? >> gpurun_out/final_smoke.txt
python bench.py --steps 20 --warmup 5 > gpurun_out/final_c5.json 2> gpurun_out/final_c5.err
for c in c1 c2 c3 c4; do python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/final_$c.json 2> gpurun_out/final_$c.err; done
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 1 --steps 5 --warmup 3 > gpurun_out/final_torchrun1.json 2> gpurun_out/final_torchrun1.err
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/final_ref.json 2>&1
echo done
