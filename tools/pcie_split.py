import json, time, torch
n = 8 * 10**9
h1 = torch.empty(n, dtype=torch.uint8, pin_memory=True); h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d1 = torch.empty(n, dtype=torch.uint8, device="cuda"); d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
S = [torch.cuda.Stream() for _ in range(4)]
def run(ups, downs):
    # ups / downs: number of streams splitting each 8 GB transfer
    evs = []
    torch.cuda.synchronize()
    t = time.perf_counter()
    k = 0
    for i in range(ups):
        a, b = i * n // ups, (i + 1) * n // ups
        with torch.cuda.stream(S[k]): d1[a:b].copy_(h1[a:b], non_blocking=True)
        k += 1
    for i in range(downs):
        a, b = i * n // downs, (i + 1) * n // downs
        with torch.cuda.stream(S[k]): h2[a:b].copy_(d2[a:b], non_blocking=True)
        k += 1
    torch.cuda.synchronize()
    return 2 * n / (time.perf_counter() - t) / 1e9
out = {}
for ups, downs in [(1, 1), (1, 2), (2, 2), (1, 3), (2, 1)]:
    run(ups, downs)
    out[f"{ups}up_{downs}down"] = round(sum(run(ups, downs) for _ in range(3)) / 3, 2)
print(json.dumps(out))
