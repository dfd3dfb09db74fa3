"""Dev utility: PCIe copy patterns at the C2a size (203 MB each way), pinned host."""
import torch
B = 256
n1, m1 = 513, 129
dev = torch.device("cuda", 0)
x = torch.randn(B, n1, m1, 3).pin_memory()
y = torch.empty(B, n1, m1, 3).pin_memory()
dx = torch.empty(B, n1, m1, 3, device=dev)
dy = torch.randn(B, n1, m1, 3, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(f, reps=8):
    ts = []
    for it in range(reps + 2):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur); s2.wait_stream(cur)
        f()
        cur.wait_stream(s1); cur.wait_stream(s2)
        e1.record(); torch.cuda.synchronize()
        if it >= 2:
            ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


def whole():
    with torch.cuda.stream(s1):
        dx.copy_(x, non_blocking=True)
    with torch.cuda.stream(s2):
        y.copy_(dy, non_blocking=True)


def chunked(c):
    def f():
        lo = 0
        for sz in c:
            hi = lo + sz
            with torch.cuda.stream(s1):
                dx[lo:hi].copy_(x[lo:hi], non_blocking=True)
            with torch.cuda.stream(s2):
                y[lo:hi].copy_(dy[lo:hi], non_blocking=True)
            lo = hi
    return f


def h2d_only():
    with torch.cuda.stream(s1):
        dx.copy_(x, non_blocking=True)


def d2h_only():
    with torch.cuda.stream(s2):
        y.copy_(dy, non_blocking=True)


print("H2D only      %.3f ms" % timed(h2d_only))
print("D2H only      %.3f ms" % timed(d2h_only))
print("whole both    %.3f ms" % timed(whole))
print("chunked 32x8  %.3f ms" % timed(chunked([32] * 8)))
print("chunked 8x32  %.3f ms" % timed(chunked([8] * 32)))

s3, s4 = torch.cuda.Stream(), torch.cuda.Stream()


def chunked2(c):
    """two copy streams per direction, chunks alternating"""
    def f():
        cur = torch.cuda.current_stream()
        s3.wait_stream(cur); s4.wait_stream(cur)
        lo = 0
        for k, sz in enumerate(c):
            hi = lo + sz
            with torch.cuda.stream(s1 if k % 2 == 0 else s3):
                dx[lo:hi].copy_(x[lo:hi], non_blocking=True)
            with torch.cuda.stream(s2 if k % 2 == 0 else s4):
                y[lo:hi].copy_(dy[lo:hi], non_blocking=True)
            lo = hi
        cur.wait_stream(s3); cur.wait_stream(s4)
    return f


print("chunked2 32x8 %.3f ms" % timed(chunked2([32] * 8)))
print("chunked2 16x16 %.3f ms" % timed(chunked2([16] * 16)))
