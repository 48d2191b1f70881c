import os,sys,torch
sys.path.insert(0,'.')
os.environ['MXFFT_B200_LIB']=os.path.abspath('paper_2512_04317_b200/_lib_pst/libmxfft_b200.so')
import paper_2512_04317_b200 as mx
from paper_2512_04317_b200.workloads import ellipse_kspace_batch
n=int(sys.argv[1]) if len(sys.argv)>1 else 256; b=int(sys.argv[2]) if len(sys.argv)>2 else 256
x=torch.from_numpy(ellipse_kspace_batch(b,n,seed=0)).cuda()
for i in range(3):
    mx.prescale_stats_device(x,b,n*n,mx.PrescaleConfig()); torch.cuda.synchronize()
