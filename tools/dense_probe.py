import sys, os; sys.path.insert(0, os.getcwd())
import torch, paper_1610_06209_b200 as spn
sp = spn.StackedSpinner(spn.SpinnerVariant.gaussian_dense, 1024, 1024, 4096, 5)
x = torch.randn(4096, 1024, device="cuda")
for _ in range(3): y = sp.apply(x)
torch.cuda.synchronize(); print("ok")
