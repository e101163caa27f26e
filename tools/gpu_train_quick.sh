mkdir -p gpurun_out
for m in host device graph; do timeout 300 python tools/probe_train.py 4096 2000 $m >> gpurun_out/tq_probe.log 2>&1; done
timeout 300 python tools/probe_train.py 4096 10000 graph >> gpurun_out/tq_probe.log 2>&1
timeout 300 python -c "
import sys,time,torch; sys.path.insert(0,'.')
from paper_2401_07886_b200 import default_tiers, RewardSpec
from paper_2401_07886_b200.trainer import TrainConfig, DeviceLearner
from paper_2401_07886_b200.env import EnvBatch
for i in range(3):
    torch.cuda.synchronize(); t0=time.time()
    L=DeviceLearner(4,3,TrainConfig(batch_size=512, buffer_capacity=1<<20),4096,4096)
    torch.cuda.synchronize(); t1=time.time()
    e=EnvBatch(default_tiers(), RewardSpec.default(), 4096, None, ring_capacity=1024)
    torch.cuda.synchronize(); t2=time.time()
    L.close(); e.close(); torch.cuda.synchronize(); t3=time.time()
    print('learner create',t1-t0,'env create',t2-t1,'close',t3-t2)
" >> gpurun_out/tq_probe.log 2>&1
