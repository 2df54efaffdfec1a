import torch, torch.nn.functional as F
dev="cuda"
P,V,B,l=4096,64,64,40
emit=torch.randn(P,V,device=dev)
tok=torch.randint(0,V,(B,l),device=dev)
dun=torch.randn(B,l,P,device=dev)
def t(f,n=50):
    for _ in range(5): f()
    e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(n): f()
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1)/n*1e3
print("gather strided   %.1f us"%t(lambda: emit.t()[tok].contiguous()))
print("gather contig    %.1f us"%t(lambda: emit.t().contiguous()[tok]))
print("embedding        %.1f us"%t(lambda: F.embedding(tok, emit.t().contiguous())))
print("index_add        %.1f us"%t(lambda: torch.zeros(V,P,device=dev).index_add_(0,tok.view(-1),dun.reshape(-1,P))))
oh=lambda: F.one_hot(tok.view(-1),V).float()
print("onehot mm        %.1f us"%t(lambda: oh().t() @ dun.reshape(-1,P)))
a=torch.zeros(V,P,device=dev).index_add_(0,tok.view(-1),dun.reshape(-1,P)); b=oh().t() @ dun.reshape(-1,P)
print("max diff", (a-b).abs().max().item(), a.abs().max().item())
# autograd path of the train step: gather + backward
le=emit.clone().requires_grad_(True)
def fb():
    u=le.t()[tok]; g,=torch.autograd.grad(u, le, dun); return g
def fb2():
    u=F.embedding(tok, le.t().contiguous()); g,=torch.autograd.grad(u, le, dun); return g
print("autograd strided %.1f us"%t(fb,20))
print("autograd embed   %.1f us"%t(fb2,20))
