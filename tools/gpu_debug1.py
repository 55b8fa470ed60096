import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import numpy as np, torch, oracle
from helpers import residuals
import paper_1205_2107_b200 as P
from paper_1205_2107_b200 import workloads as W
d,e=W.random_uniform(50,0)
dt=torch.tensor(d,device='cuda'); et=torch.tensor(e,device='cuda')
w,Z=P.stemr(dt,et); w=w.cpu().numpy(); Z=Z.cpu().numpy()
wo,Zo=oracle.stemr(d,e)
rg=residuals(d,e,w,Z); rgo=residuals(d,e,wo,Z)
for j in range(50):
    print(j, "%.17g %.17g diff=%.3e resid(own w)=%.2e resid(oracle w)=%.2e"%(w[j],wo[j],w[j]-wo[j],rg[j],rgo[j]))
