for i in 1 2 3; do timeout 300 python tools/determinism_probe.py --case c2 --configs 0 --runs 1 --save gpurun_out/det_p$i.npy > /dev/null 2>&1; done
python -c "
import numpy as np
a=[np.load(f'gpurun_out/det_p{i}.npy') for i in (1,2,3)]
print('cross-process', [[float(np.abs(a[i][s]-a[0][s]).max()) for s in range(4)] for i in (1,2)])
"
CUDA_LAUNCH_BLOCKING=1 timeout 600 python tools/determinism_probe.py --case c2 --configs 0,1 --runs 3
