// Gmsh 2.2 ASCII mesh reader (load_mesh, /root/reference/pkg/src/hbem/mesh.py:134-245).
//
// Same acceptance rules, section handling, error wording and line numbers as
// the reference parser:
//   * lines are split like str.splitlines(), tokens like str.split();
//   * $MeshFormat: version must start with "2.", file type must be "0"
//     (ASCII); $EndMeshFormat is not required (unknown lines are skipped);
//   * $Nodes / $Elements: a count line, then exactly that many records, then
//     the closing tag; node tags may repeat (the last one wins);
//   * only 3-node triangles (type 2) become elements, every other element is
//     counted as skipped; referenced vertices are compacted in ascending tag
//     order and element indices renumbered accordingly.
// Numbers are parsed with the C library (strtod is correctly rounded, as is
// Python's float(), so coordinates are bit-identical).  Big meshes (millions of
// triangles) parse in a fraction of a second instead of the reference's
// per-line Python loop.
#include <algorithm>
#include <array>
#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/hbem_b200.h"

namespace hb {
int set_error(int code, const char *fmt, ...);
void clear_error();
}  // namespace hb

struct hbem_mesh_file {
  std::vector<double> vertices;   // nv x 3
  std::vector<int64_t> elements;  // m x 3
  int64_t skipped = 0;
};

namespace {

thread_local int64_t g_err_line = -1;
thread_local char g_err_section[32] = {0};

struct Line {
  const char *b, *e;
};

inline bool is_ws(char c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\v' || c == '\f' ||
         (c >= '\x1c' && c <= '\x1f');
}

// str.splitlines(): \n, \r, \r\n, \v, \f, \x1c, \x1d, \x1e
std::vector<Line> split_lines(const std::string &s) {
  std::vector<Line> out;
  const char *p = s.data(), *end = p + s.size(), *b = p;
  while (p < end) {
    const char c = *p;
    if (c == '\n' || c == '\r' || c == '\v' || c == '\f' || c == '\x1c' || c == '\x1d' ||
        c == '\x1e') {
      out.push_back({b, p});
      if (c == '\r' && p + 1 < end && p[1] == '\n') ++p;
      b = p + 1;
    }
    ++p;
  }
  if (b < end) out.push_back({b, end});
  return out;
}

std::vector<std::string> tokens(const Line &l) {
  std::vector<std::string> out;
  const char *p = l.b;
  while (p < l.e) {
    while (p < l.e && is_ws(*p)) ++p;
    const char *b = p;
    while (p < l.e && !is_ws(*p)) ++p;
    if (p > b) out.emplace_back(b, p);
  }
  return out;
}

std::string stripped(const Line &l) {
  const char *b = l.b, *e = l.e;
  while (b < e && is_ws(*b)) ++b;
  while (e > b && is_ws(e[-1])) --e;
  return std::string(b, e);
}

// int(token): optional sign, decimal digits (single underscores between
// digits allowed, as Python accepts them)
bool parse_int(std::string t, long long &v) {
  if (t.empty()) return false;
  std::string s;
  for (size_t i = 0; i < t.size(); ++i) {
    if (t[i] == '_') {
      if (i == 0 || i + 1 == t.size() || !isdigit((unsigned char)t[i - 1]) ||
          !isdigit((unsigned char)t[i + 1]))
        return false;
      continue;
    }
    s += t[i];
  }
  size_t i = (s[0] == '+' || s[0] == '-') ? 1 : 0;
  if (i == s.size()) return false;
  for (size_t j = i; j < s.size(); ++j)
    if (!isdigit((unsigned char)s[j])) return false;
  errno = 0;
  char *end = nullptr;
  v = std::strtoll(s.c_str(), &end, 10);
  return errno == 0 && *end == '\0';
}

// float(token): decimal literal, inf/nan spellings; no hexadecimal (Python's
// float() rejects it, strtod would accept it)
bool parse_float(const std::string &t, double &v) {
  if (t.empty()) return false;
  for (char c : t)
    if (c == 'x' || c == 'X' || c == 'p' || c == 'P') return false;
  std::string s;
  for (size_t i = 0; i < t.size(); ++i)
    if (t[i] != '_') s += t[i];
    else if (i == 0 || i + 1 == t.size() || !isdigit((unsigned char)t[i - 1]) ||
             !isdigit((unsigned char)t[i + 1]))
      return false;
  char *end = nullptr;
  v = std::strtod(s.c_str(), &end);
  return end != s.c_str() && *end == '\0';
}

int parse_error(const char *name, const char *msg, long long line, const char *section) {
  g_err_line = line;
  std::snprintf(g_err_section, sizeof(g_err_section), "%s", section ? section : "");
  std::string loc;
  if (section) loc += std::string("section ") + section;
  if (line >= 0) {
    if (!loc.empty()) loc += ", ";
    loc += "line " + std::to_string(line);
  }
  if (loc.empty()) return hb::set_error(HBEM_ERR_MESH_PARSE, "%s: %s", name, msg);
  return hb::set_error(HBEM_ERR_MESH_PARSE, "%s: %s (%s)", name, msg, loc.c_str());
}

}  // namespace

extern "C" {

int hbem_gmsh_read(const char *path, hbem_mesh_file **out) {
  hb::clear_error();
  g_err_line = -1;
  g_err_section[0] = 0;
  if (!path || !out) return hb::set_error(HBEM_ERR_ARG, "null argument");
  *out = nullptr;
  const char *slash = std::strrchr(path, '/');
  const char *name = slash ? slash + 1 : path;
  std::string text;
  {
    FILE *f = std::fopen(path, "rb");
    if (!f)
      return hb::set_error(HBEM_ERR_MESH, "cannot read mesh file %s: [Errno %d] %s: '%s'", path,
                           errno, std::strerror(errno), path);
    char buf[1 << 16];
    size_t n;
    while ((n = std::fread(buf, 1, sizeof(buf), f)) > 0) text.append(buf, n);
    const bool bad = std::ferror(f);
    std::fclose(f);
    if (bad) return hb::set_error(HBEM_ERR_MESH, "cannot read mesh file %s: read error", path);
  }
  const std::vector<Line> lines = split_lines(text);
  const long long n = (long long)lines.size();
  std::unordered_map<long long, std::array<double, 3>> nodes;
  std::vector<long long> tri;
  long long skipped = 0;
  bool saw_format = false, saw_nodes = false, saw_elements = false;
  long long i = 0;
  char msg[256];
  while (i < n) {
    const std::string tok = stripped(lines[i]);
    if (tok == "$MeshFormat") {
      const std::vector<std::string> header = i + 1 < n ? tokens(lines[i + 1]) : std::vector<std::string>();
      if (header.empty()) return parse_error(name, "missing format line", i + 2, "$MeshFormat");
      if (header[0].compare(0, 2, "2.") != 0) {
        std::snprintf(msg, sizeof(msg), "unsupported format version '%s', expected 2.x ASCII",
                      header[0].c_str());
        return parse_error(name, msg, i + 2, "$MeshFormat");
      }
      if (header.size() > 1 && header[1] != "0")
        return parse_error(name, "binary files are not supported", i + 2, "$MeshFormat");
      saw_format = true;
      i += 2;
    } else if (tok == "$Nodes") {
      saw_nodes = true;
      long long count = 0;
      if (i + 1 >= n || !parse_int(stripped(lines[i + 1]), count))
        return parse_error(name, "expected node count", i + 2, "$Nodes");
      nodes.reserve((size_t)std::max(count, 0ll));
      for (long long k = 0; k < count; ++k) {
        const long long ln = i + 2 + k;
        long long tag;
        std::array<double, 3> xyz;
        bool ok = ln < n;
        if (ok) {
          const std::vector<std::string> p = tokens(lines[ln]);
          ok = p.size() >= 4 && parse_int(p[0], tag) && parse_float(p[1], xyz[0]) &&
               parse_float(p[2], xyz[1]) && parse_float(p[3], xyz[2]);
        }
        if (!ok) return parse_error(name, "malformed node line", ln + 1, "$Nodes");
        nodes[tag] = xyz;
      }
      i += 2 + std::max(count, 0ll);
      if (i >= n || stripped(lines[i]) != "$EndNodes")
        return parse_error(name, "missing $EndNodes", i + 1, "$Nodes");
      ++i;
    } else if (tok == "$Elements") {
      saw_elements = true;
      long long count = 0;
      if (i + 1 >= n || !parse_int(stripped(lines[i + 1]), count))
        return parse_error(name, "expected element count", i + 2, "$Elements");
      for (long long k = 0; k < count; ++k) {
        const long long ln = i + 2 + k;
        std::vector<long long> p;
        bool ok = ln < n;
        if (ok) {
          for (const std::string &t : tokens(lines[ln])) {
            long long v;
            if (!parse_int(t, v)) { ok = false; break; }
            p.push_back(v);
          }
        }
        ok = ok && p.size() >= 3;
        if (!ok) return parse_error(name, "malformed element line", ln + 1, "$Elements");
        const long long etype = p[1], ntags = p[2];
        const long long c0 = 3 + ntags;
        if (etype == 2) {
          const long long nc = c0 < 0 ? 0 : std::max(0ll, (long long)p.size() - c0);
          if (c0 < 0 || nc != 3) {
            std::snprintf(msg, sizeof(msg), "triangle with %lld nodes",
                          c0 < 0 ? (long long)p.size() : nc);
            return parse_error(name, msg, ln + 1, "$Elements");
          }
          tri.push_back(p[c0]);
          tri.push_back(p[c0 + 1]);
          tri.push_back(p[c0 + 2]);
        } else {
          ++skipped;
        }
      }
      i += 2 + std::max(count, 0ll);
      if (i >= n || stripped(lines[i]) != "$EndElements")
        return parse_error(name, "missing $EndElements", i + 1, "$Elements");
      ++i;
    } else {
      ++i;
    }
  }
  if (!saw_format) return parse_error(name, "no $MeshFormat section", -1, nullptr);
  if (!saw_nodes) return parse_error(name, "no $Nodes section", -1, nullptr);
  if (!saw_elements) return parse_error(name, "no $Elements section", -1, nullptr);
  if (tri.empty()) return parse_error(name, "file contains no triangles", -1, nullptr);
  std::vector<long long> used(tri);
  std::sort(used.begin(), used.end());
  used.erase(std::unique(used.begin(), used.end()), used.end());
  hbem_mesh_file *m = new (std::nothrow) hbem_mesh_file;
  if (!m) return hb::set_error(HBEM_ERR_CAPACITY, "out of host memory");
  m->vertices.resize(used.size() * 3);
  for (size_t j = 0; j < used.size(); ++j) {
    auto it = nodes.find(used[j]);
    if (it == nodes.end()) {
      delete m;
      std::snprintf(msg, sizeof(msg), "element references unknown node tag %lld", used[j]);
      return parse_error(name, msg, -1, nullptr);
    }
    for (int c = 0; c < 3; ++c) m->vertices[3 * j + c] = it->second[c];
  }
  m->elements.resize(tri.size());
  for (size_t j = 0; j < tri.size(); ++j)
    m->elements[j] = std::lower_bound(used.begin(), used.end(), tri[j]) - used.begin();
  m->skipped = skipped;
  *out = m;
  return HBEM_OK;
}

int hbem_gmsh_size(const hbem_mesh_file *m, int64_t *n_vertices, int64_t *n_elements,
                   int64_t *n_skipped) {
  if (!m || !n_vertices || !n_elements || !n_skipped)
    return hb::set_error(HBEM_ERR_ARG, "null argument");
  *n_vertices = (int64_t)m->vertices.size() / 3;
  *n_elements = (int64_t)m->elements.size() / 3;
  *n_skipped = m->skipped;
  return HBEM_OK;
}

int hbem_gmsh_copy(const hbem_mesh_file *m, double *vertices, int64_t *elements) {
  if (!m || !vertices || !elements) return hb::set_error(HBEM_ERR_ARG, "null argument");
  std::memcpy(vertices, m->vertices.data(), m->vertices.size() * sizeof(double));
  std::memcpy(elements, m->elements.data(), m->elements.size() * sizeof(int64_t));
  return HBEM_OK;
}

int hbem_gmsh_error_location(int64_t *line, char *section, int32_t cap) {
  if (!line || !section || cap < 1) return hb::set_error(HBEM_ERR_ARG, "null argument");
  *line = g_err_line;
  std::snprintf(section, (size_t)cap, "%s", g_err_section);
  return HBEM_OK;
}

int hbem_gmsh_destroy(hbem_mesh_file *m) {
  delete m;
  return HBEM_OK;
}

}  // extern "C"
