"""A literal CELF over fixed sketches: the reference count of
re-evaluations for the library's CELF counter (PACIM_CELF_COUNT).  Test
infrastructure (pure Python, tiny inputs)."""


def celf_reevaluations(labs, sizes, n, k):
    """CELF literally, with a heap of (stale score desc, id asc):
    marginal gains recomputed from the sketches' labels (the oracle's), the
    re-evaluations from step 2 on counted (step 1 reads the initial, fresh
    scores).  Returns (seeds, gains, re-evaluations)."""
    import heapq
    R = len(labs)
    covered = [set() for _ in range(R)]

    def gain(v):
        return sum(int(sizes[r][v]) for r in range(R) if labs[r][v] not in covered[r])

    heap = [(-gain(v), v, 0) for v in range(n)]  # (-score, id, step of the evaluation)
    heapq.heapify(heap)
    seeds, gains, reev = [], [], 0
    for step in range(k):
        while True:
            negg, v, st = heapq.heappop(heap)
            if st == step:
                break
            reev += 1
            heapq.heappush(heap, (-gain(v), v, step))
        seeds.append(v)
        gains.append(-negg)
        for r in range(R):
            covered[r].add(labs[r][v])
    return seeds, gains, reev
